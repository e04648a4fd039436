// gf_graph.cu -- device block store: create/grow, batch append (K1), deletes, exports.
//
// K1 replaces DynamicGraph.add_edges / _append_edge / node_t_max
// (reference storage.py:382-477).  The reference appends edge by edge; here a
// whole batch is appended with sorts and scans, reproducing the reference's
// state exactly (same block handles, capacities, links, slot order, ids):
//   events (edge j, endpoint side) -> stable radix sort by node -> per-node
//   segments -> chronology check (serial resolve only if a batch could reject)
//   -> ids by scan -> per-segment block plan (capacity law with the live
//   degree at allocation) -> handles and slot bases by one scan over the events
//   that trigger an allocation (= the reference's allocation order; handles
//   freed by offload are reused LIFO first) -> metadata/directory/slot writes.
// Nothing is read back mid-call (see add_edges_fast), and the launch sequence
// is replayed as a CUDA graph.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <string.h>

#include <algorithm>
#include <chrono>
#include <tuple>
#include <vector>

#include "gf_graph.cuh"

using namespace gf;
namespace cg = cooperative_groups;

namespace {

// staged batch: one 32-byte record per edge {src, dst, ts, eid} -- after the sort by node every
// per-event access is a random access by edge index, and one record is one sector (separate
// src/dst/ts/eid arrays cost a random line each at 10M-edge batches)
constexpr int ER = 4, ER_SRC = 0, ER_DST = 1, ER_TS = 2, ER_EID = 3;

struct IngestCounters {
  long long minv, maxv;   // node id range of the batch
  long long viol;         // 1 if the batch may reject an edge
  long long num_segs;     // distinct stored endpoints
  long long n_acc;        // accepted edges
  long long new_blocks;   // blocks to allocate
  long long new_slots;    // slots to allocate
  long long dir_need;     // directory entries to allocate
  long long max_eid;      // max preassigned accepted id
  long long abort;        // sync-free path: ABORT_* bits, nothing was mutated
  long long tsmin, tsmax; // timestamp range of the batch (32-bit fence validity)
  long long num_big;      // cooperative path: segments with more than 32 events
  long long num_moves;    // cooperative path: directories that move to a larger region
  long long phase_ns[12]; // cooperative path: globaltimer at each phase start (GF_INGEST_TIMING)
  long long done;         // cooperative path: CTAs finished (the last one publishes and re-arms)
};

// the values every call starts from
__host__ __device__ inline void counters_arm(IngestCounters* c) {
  long long* w = reinterpret_cast<long long*>(c);
  for (size_t i = 0; i < sizeof(IngestCounters) / sizeof(long long); i++) w[i] = 0;
  c->minv = c->tsmin = LLONG_MAX;
  c->maxv = c->tsmax = c->max_eid = LLONG_MIN;
}
// ABORT_SLOW (cooperative path only): the batch needs the general launch sequence -- an endpoint
// may see a decreasing timestamp (possible rejection), or a segment exceeds what one CTA sorts
constexpr long long ABORT_NODES = 1, ABORT_CAP = 2, ABORT_SLOW = 4;

// per-call values of the sync-free path, read on the device so that its captured launch
// sequence can be replayed unchanged (one H2D copy of this struct per call)
struct IngestScalars {
  const int64_t *src, *dst, *ts, *eids_in;
  int64_t* out_eids;
  int64_t num_nodes, blk_used, slots_used, dir_used, next_edge_id, slots_free, dir_free;
  const int64_t* free_list;  // handles freed by offload, reused LIFO (storage.py:171-181)
  int64_t nfree;
  int64_t blocks_free;       // cooperative path: block-arena capacity left (checked on the device)
};

template <class T>
gf_status grow_array(T*& p, int64_t keep, int64_t new_cap, cudaStream_t s) {
  T* q = nullptr;
  cudaError_t e = cudaMallocAsync(&q, sizeof(T) * (size_t)std::max<int64_t>(new_cap, 1), s);
  if (e != cudaSuccess) return fail(GF_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e));
  if (p && keep > 0) GF_CUDA(cudaMemcpyAsync(q, p, sizeof(T) * (size_t)keep, cudaMemcpyDeviceToDevice, s));
  if (p) cudaFreeAsync(p, s);
  p = q;
  return GF_OK;
}



// one event per (edge, stored endpoint), in the reference's append order
__global__ void k_make_events(const int64_t* __restrict__ rec, int64_t n, int directed, uint32_t* keys, uint32_t* vals,
                              const IngestCounters* c, longlong2* trig) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  int64_t E = directed ? n : 2 * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = directed ? e : (e >> 1);
    int side = directed ? 0 : (int)(e & 1);
    keys[e] = (uint32_t)rec[ER * j + (side ? ER_DST : ER_SRC)];
    vals[e] = (uint32_t)e;
    if (trig) trig[e] = make_longlong2(0, 0);
  }
}

__device__ __forceinline__ int64_t ev_edge(uint32_t ev, int directed) { return directed ? (int64_t)ev : (int64_t)(ev >> 1); }

__device__ __forceinline__ int64_t node_tmax(const int64_t* tail, const int64_t* bsize, const int64_t* btmax, int64_t v) {
  int64_t t = tail[v];
  if (t == GF_NO_BLOCK || bsize[t] == 0) return GF_TS_MIN;  // storage.py:382-390
  return btmax[t];
}

__global__ void k_heads(const uint32_t* __restrict__ keys, int64_t E, int32_t* heads) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x)
    heads[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// seg_id = inclusive_scan(heads) - 1; record segment starts, detect possible rejections
__global__ void k_segments(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, const int32_t* __restrict__ incl,
                           int64_t E, int directed, const int64_t* __restrict__ rec, const int64_t* tail, const int64_t* bsize,
                           const int64_t* btmax, int64_t* seg_start, IngestCounters* c) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = incl[i] - 1;
    bool head = (i == 0) || keys[i] != keys[i - 1];
    int64_t t = rec[ER * ev_edge(vals[i], directed) + ER_TS];
    bool viol;
    if (head) {
      seg_start[s] = i;
      viol = t < node_tmax(tail, bsize, btmax, keys[i]);
    } else {
      viol = t < rec[ER * ev_edge(vals[i - 1], directed) + ER_TS];
    }
    if (viol) atomicOr((unsigned long long*)&c->viol, 1ull);
    if (i == E - 1) c->num_segs = s + 1;
  }
}






// compacted accepted events (segment-major, arrival order inside a segment)
__global__ void k_compact(const uint32_t* __restrict__ vals, const int32_t* __restrict__ incl, const int64_t* __restrict__ cpos,
                          const int64_t* __restrict__ keep, const int64_t* __restrict__ seg_start, int64_t E,
                          const IngestCounters* c, uint32_t* ce_ev, int64_t* ce_pend, int32_t* ce_seg) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  int64_t nseg = c->num_segs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    int32_t s = incl[i] - 1;
    int64_t end = (s + 1 < nseg) ? seg_start[s + 1] : E;
    int64_t p = cpos[i];
    ce_ev[p] = vals[i];
    ce_pend[p] = end - i;  // pending count incl. later rejected events (storage.py:417-447)
    ce_seg[p] = s;
  }
}

__device__ __forceinline__ int64_t sizing_cap(int kind, int64_t tau, int64_t param, int64_t degree, int64_t pending) {
  if (kind == GF_SIZING_FIXED) return param;                // storage.py:102-103
  if (kind == GF_SIZING_BATCH) return pending > 1 ? pending : 1;  // storage.py:116-117
  int64_t d = degree > 1 ? degree : 1;                      // storage.py:88-89
  return d < tau ? d : tau;
}

struct SegPlan {
  int64_t* acc_cnt;   // accepted events per segment
  int64_t* cstart;    // start in the compacted event list
  int64_t* fill;      // events that go into the current tail
  int64_t* tail_size; // tail size before the batch
  int64_t* nb_new;    // new blocks
  longlong4* plan4;   // {new blocks, new slots, new directory capacity, 0} per segment, zero to E (scan input)
};


__global__ void k_plan(const uint32_t* __restrict__ keys, const int64_t* __restrict__ seg_start,
                       const int64_t* __restrict__ cpos, const int64_t* __restrict__ ce_pend, int64_t E,
                       const IngestCounters* c, const int64_t* tail, const int64_t* bsize, const int64_t* bcap,
                       const int64_t* degree, const int64_t* num_blocks, const int64_t* dir_cap, int kind, int64_t tau,
                       int64_t param, SegPlan P, int64_t* old_tail) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  const int64_t nseg = c->num_segs;
  // the per-segment plan scan covers num_segs + 1 entries: only the last needs a zero
  if (blockIdx.x == 0 && threadIdx.x == 0) P.plan4[nseg] = make_longlong4(0, 0, 0, 0);
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t st = seg_start[s], en = (s + 1 < nseg) ? seg_start[s + 1] : E;
    int64_t cs = cpos[st], cnt = cpos[en] - cs;
    int64_t v = keys[st];
    P.acc_cnt[s] = cnt;
    P.cstart[s] = cs;
    int64_t t = tail[v];
    old_tail[s] = t;
    int64_t fill = 0, tsz = 0;
    if (t != GF_NO_BLOCK) {
      tsz = bsize[t];
      fill = min(bcap[t] - tsz, cnt);
    }
    P.fill[s] = fill;
    P.tail_size[s] = tsz;
    int64_t deg = degree[v] + fill, rem = cnt - fill, used = fill, blocks = 0, slots = 0;
    while (rem > 0) {
      int64_t cap = sizing_cap(kind, tau, param, deg, ce_pend[cs + used]);
      int64_t take = min(cap, rem);
      blocks++;
      slots += cap;
      deg += take;
      used += take;
      rem -= take;
    }
    P.nb_new[s] = blocks;
    int64_t need = num_blocks[v] + blocks;
    int64_t dc = dir_cap[v], dnew = 0;
    if (need > dc) {
      dnew = 8;
      while (dnew < need) dnew <<= 1;
    }
    P.plan4[s] = make_longlong4(blocks, slots, dnew, 0);
  }
}



struct Recs {
  int64_t* first;   // segment-local accepted rank of the block's first event
  int64_t* count;   // events placed in the block
  int64_t* cap;     // capacity
  int32_t* seg;     // owning segment
  uint32_t* key;    // original event index of the first event = allocation order
};



struct BlockArrays {
  int64_t *cap, *size, *tmin, *tmax, *prev, *next, *base;
};


struct NodeArrays {
  int64_t *head, *tail, *num_blocks, *degree, *nslots, *dir_off, *dir_cap;
  const uint8_t* valid;
  uint8_t* nflags;
  int64_t* nrec;
};
struct DirArrays {
  int64_t* e;  // DIRW words per entry
};


__global__ void k_noderec_invalidate(int64_t* nrec, int64_t v) { nrec[v * NREC + 2] &= ~NREC_VALID; }



template <class F>
gf_status cub_call(F f, cudaStream_t s) {
  size_t bytes = 0;
  GF_CUDA(f((void*)nullptr, bytes));
  Scratch tmp(s);
  GF_TRY(tmp.alloc(bytes));
  GF_CUDA(f(tmp.p, bytes));
  return GF_OK;
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 32 && ((int64_t)1 << b) < n) b++;
  return b;
}


gf_status ensure_blocks(gf_graph* g, int64_t need, cudaStream_t s) {
  if (need <= g->blk_cap) return GF_OK;
  g->gen++;
  int64_t nc = std::max<int64_t>(need, std::max<int64_t>(1024, g->blk_cap * 2));
  int64_t k = g->blk_used;
  GF_TRY(grow_array(g->bcap, k, nc, s));
  GF_TRY(grow_array(g->bsize, k, nc, s));
  GF_TRY(grow_array(g->btmin, k, nc, s));
  GF_TRY(grow_array(g->btmax, k, nc, s));
  GF_TRY(grow_array(g->bprev, k, nc, s));
  GF_TRY(grow_array(g->bnext, k, nc, s));
  GF_TRY(grow_array(g->bbase, k, nc, s));
  g->blk_cap = nc;
  return GF_OK;
}

gf_status ensure_slots(gf_graph* g, int64_t need, cudaStream_t s) {
  if (need <= g->slot_cap) return GF_OK;
  g->gen++;
  int64_t nc = std::max<int64_t>(need, std::max<int64_t>(4096, g->slot_cap + g->slot_cap / 2));
  int64_t old = g->slot_cap;
  GF_TRY(grow_array(g->slots, g->slots_used, nc, s));
  GF_TRY(grow_array(g->sts, g->slots_used, nc + 2 * FENCE, s));  // window loads may read past the end
  GF_TRY(grow_array(g->fts, (g->slots_used + FENCE - 1) / FENCE, nc / FENCE + 8, s));  // chunk loads read up to 3 past
  GF_TRY(grow_array(g->sts32, g->slots_used, nc + 2 * FENCE32, s));  // whole aligned lines are read
  GF_TRY(grow_array(g->fts32, (g->slots_used + FENCE32 - 1) / FENCE32, nc / FENCE32 + 16, s));  // chunk loads read up to 7 past
  // unused capacity slots must read as invalid (delete scans the whole pool)
  GF_CUDA(cudaMemsetAsync(g->slots + old, 0, sizeof(Slot) * (size_t)(nc - old), s));
  if (g->okbits) {
    const int64_t w_old = (old + 31) / 32, w_new = (nc + 31) / 32 + 4;  // padded: 64-bit runs read 3 words
    GF_TRY(grow_array(g->okbits, w_old, w_new, s));
    GF_CUDA(cudaMemsetAsync(g->okbits + w_old, 0, sizeof(uint32_t) * (size_t)(w_new - w_old), s));
  }
  g->slot_cap = nc;
  return GF_OK;
}

gf_status ensure_dir(gf_graph* g, int64_t need, cudaStream_t s) {
  if (need <= g->dir_cap_total) return GF_OK;
  g->gen++;
  int64_t nc = std::max<int64_t>(need, std::max<int64_t>(4096, g->dir_cap_total * 2));
  GF_TRY(grow_array(g->dir, g->dir_used * DIRW, nc * DIRW, s));
  g->dir_cap_total = nc;
  return GF_OK;
}


// ---- sync-free ingest --------------------------------------------------------
// The same plan as add_edges_impl, but every size the host needs is either bounded by the
// batch (new blocks <= events) or checked on the device: node-table growth beyond the
// capacity and slot/directory pool overflow set IngestCounters.abort before anything is
// mutated, and the host grows the pools and replays the batch.  Block handles and slot bases
// come from one scan over the events that trigger an allocation (allocation order =
// triggering event order), so there is no sort over new blocks and no mid-call host sync:
// one launch sequence, one synchronisation at the end (for the rejected count).


// node-table growth on the device: rows [lo, maxv + 1) when they fit the capacity
__global__ void k_grow_nodes(IngestCounters* c, const IngestScalars* S, int64_t cap, int64_t* head, int64_t* tail,
                             int64_t* nb, int64_t* deg, uint8_t* valid, int64_t* nslots, int64_t* doff, int64_t* dcap,
                             uint8_t* nflags, int64_t* nrec) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  const int64_t lo = S->num_nodes;
  const long long hi = c->maxv + 1;
  if (c->minv < 0 || hi > cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) c->abort |= ABORT_NODES;
    return;
  }
  for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi; v += (int64_t)gridDim.x * blockDim.x) {
    head[v] = GF_NO_BLOCK;
    tail[v] = GF_NO_BLOCK;
    nb[v] = 0;
    deg[v] = 0;
    valid[v] = 1;
    nslots[v] = 0;
    doff[v] = -1;
    dcap[v] = 0;
    nflags[v] = 0;
    int64_t* r = nrec + v * NREC;
    r[0] = -1;
    r[1] = 0;
    r[2] = NREC_VALID;
    for (int w = 3; w < NREC; w++) r[w] = 0;
  }
}

// Exclusive sum scan of K-wide int64 records (the 4-wide block plan and the 2-wide allocation
// triggers) in one pass: ticketed tiles with decoupled look-back.  Tile state (flags, ticket) is
// zeroed by k_stage_minmax at the start of the same launch sequence.
// items per thread: 4 for the latency-bound small batches, 16 for batches of >= 1M events (fewer,
// fuller tiles for the look-back chain)
constexpr int SCAN_T = 256, SCAN_ITEMS_SMALL = 4, SCAN_ITEMS_LARGE = 16;
constexpr int64_t SCAN_LARGE_EVENTS = 1 << 20;
inline int scan_tile(int64_t E) { return SCAN_T * (E >= SCAN_LARGE_EVENTS ? SCAN_ITEMS_LARGE : SCAN_ITEMS_SMALL); }

struct ScanState {
  int64_t* agg;   // [tiles][K]
  int64_t* inc;   // [tiles][K]
  int* flag;      // [tiles]: 0 none, 1 aggregate, 2 inclusive
  unsigned* ticket;
  int64_t tiles;
};

__device__ __forceinline__ int ld_flag(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_flag(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int K, int SCAN_ITEMS>
__global__ void __launch_bounds__(SCAN_T) k_scan_sum(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                                                      ScanState S, const IngestCounters* c, bool per_segment) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  __shared__ unsigned s_tile;
  __shared__ int64_t s_w[SCAN_T / 32][K];
  __shared__ int64_t s_base[K];
  if (c->abort) return;
  // per-segment records: only num_segs + 1 of the E + 1 entries can be nonzero (the last is the total)
  if (per_segment) n = min(n, (int64_t)c->num_segs + 1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(S.ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  constexpr int SCAN_TILE = SCAN_T * SCAN_ITEMS;
  if (tile * SCAN_TILE >= n) return;  // no later tile looks back at this one
  const int64_t i0 = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS][K], run[K];
#pragma unroll
  for (int f = 0; f < K; f++) run[f] = 0;
#pragma unroll
  for (int j = 0; j < SCAN_ITEMS; j++)
#pragma unroll
    for (int f = 0; f < K; f++) {
      v[j][f] = run[f];  // exclusive within the thread
      run[f] += (i0 + j < n) ? in[(i0 + j) * K + f] : 0;
    }
  // warp inclusive scan of the thread totals
  int64_t inc_[K];
#pragma unroll
  for (int f = 0; f < K; f++) {
    int64_t x = run[f];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    inc_[f] = x;
    if (lane == 31) s_w[w][f] = x;
  }
  __syncthreads();
  int64_t wpre[K], agg[K];
#pragma unroll
  for (int f = 0; f < K; f++) {
    wpre[f] = 0;
    agg[f] = 0;
#pragma unroll
    for (int i = 0; i < SCAN_T / 32; i++) {
      wpre[f] += (i < w) ? s_w[i][f] : 0;
      agg[f] += s_w[i][f];
    }
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < K; f++) (tile == 0 ? S.inc : S.agg)[tile * K + f] = agg[f];
    __threadfence();
    st_flag(S.flag + tile, tile == 0 ? 2 : 1);
  }
  if (w == 0) {
    int64_t base[K];
#pragma unroll
    for (int f = 0; f < K; f++) base[f] = 0;
    if (tile > 0) {
      int64_t end = tile - 1;
      while (true) {
        const int64_t idx = end - lane;
        int fl = 2;
        if (idx >= 0) {
          do {
            fl = ld_flag(S.flag + idx);
          } while (fl == 0);
        }
        __syncwarp();
        __threadfence();
        const unsigned incm = __ballot_sync(0xffffffffu, fl == 2);  // lanes before tile 0 count as inclusive 0
        const int first = incm ? __ffs(incm) - 1 : 31;
        const bool take = lane <= first && idx >= 0;
#pragma unroll
        for (int f = 0; f < K; f++) {
          int64_t x = take ? __ldcg((fl == 2 ? S.inc : S.agg) + idx * K + f) : 0;  // L2: never a stale L1 line
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          base[f] += x;
        }
        if (incm) break;
        end -= 32;
      }
      if (lane == 0) {
#pragma unroll
        for (int f = 0; f < K; f++) S.inc[tile * K + f] = base[f] + agg[f];
        __threadfence();
        st_flag(S.flag + tile, 2);
      }
    }
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < K; f++) s_base[f] = base[f];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < SCAN_ITEMS; j++)
    if (i0 + j < n)
#pragma unroll
      for (int f = 0; f < K; f++) out[(i0 + j) * K + f] = s_base[f] + wpre[f] + inc_[f] - run[f] + v[j][f];
}

// ---- fused kernels of the sync-free path -------------------------------------
// staging + batch min/max (the counters were initialised by the H2D copy that starts the sequence)
__global__ void k_stage_minmax(const IngestScalars* S, int64_t n, int64_t* rec, IngestCounters* c, int* zero, int64_t nzero) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nzero; j += (int64_t)gridDim.x * blockDim.x)
    zero[j] = 0;  // look-back scan flags and tickets of this launch sequence
  const bool has_eids = S->eids_in != nullptr;
  long long mn = LLONG_MAX, mx = LLONG_MIN, tn = LLONG_MAX, tx = LLONG_MIN;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const long long a = S->src[j], b = S->dst[j], t = S->ts[j];
    reinterpret_cast<longlong4*>(rec)[j] = make_longlong4(a, b, t, has_eids ? S->eids_in[j] : 0);
    mn = min(mn, min(a, b));
    mx = max(mx, max(a, b));
    tn = min(tn, t);
    tx = max(tx, t);
  }
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    tn = min(tn, __shfl_xor_sync(0xffffffffu, tn, o));
    tx = max(tx, __shfl_xor_sync(0xffffffffu, tx, o));
  }
  __shared__ long long sm[4][32];
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) {
    sm[0][w] = mn;
    sm[1][w] = mx;
    sm[2][w] = tn;
    sm[3][w] = tx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < nw; i++) {
      mn = min(mn, sm[0][i]);
      mx = max(mx, sm[1][i]);
      tn = min(tn, sm[2][i]);
      tx = max(tx, sm[3][i]);
    }
    if (mn != LLONG_MAX) {
      atomicMin(&c->minv, mn);
      atomicMax(&c->maxv, mx);
      atomicMin(&c->tsmin, tn);
      atomicMax(&c->tsmax, tx);
    }
  }
}

// chronology: accept all; only when some endpoint may see a decreasing timestamp, block 0 prepares
// the per-node latest timestamps and resolves the batch serially (storage.py:426-437)
__global__ void k_accept(uint8_t* acc, int64_t n, int64_t* tm, const int64_t* tail, const int64_t* bsize,
                         const int64_t* btmax, const IngestCounters* c, const IngestScalars* S, const int64_t* rec,
                         int directed) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  if (!c->viol) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) acc[j] = 1;
    return;
  }
  if (blockIdx.x != 0) return;
  const int64_t nn = max((int64_t)S->num_nodes, (int64_t)c->maxv + 1);
  for (int64_t v = threadIdx.x; v < nn; v += blockDim.x) tm[v] = node_tmax(tail, bsize, btmax, v);
  __syncthreads();
  if (threadIdx.x) return;
  for (int64_t j = 0; j < n; j++) {
    const int64_t a = rec[ER * j + ER_SRC], d = rec[ER * j + ER_DST], t = rec[ER * j + ER_TS];
    const bool ok = t >= tm[a] && (directed || t >= tm[d]);
    acc[j] = ok;
    if (ok) {
      tm[a] = t;
      if (!directed) tm[d] = t;
    }
  }
}

// edge ids (storage.py:438-442) and per-event keep flags in one pass
__global__ void k_eids_keep(const uint8_t* __restrict__ acc, const int64_t* __restrict__ rank, int64_t n,
                            bool has_eids, int64_t* rec, IngestCounters* c, const IngestScalars* S,
                            const uint32_t* __restrict__ vals, int64_t E, int directed, int64_t* keep) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  const int64_t next_id = S->next_edge_id;
  long long mx = LLONG_MIN;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = -1;
    if (acc[j]) {
      e = has_eids ? rec[ER * j + ER_EID] : next_id + rank[j];  // preassigned ids were staged in the record
      mx = max(mx, (long long)e);
    }
    rec[ER * j + ER_EID] = e;
    S->out_eids[j] = e;
    if (j == n - 1) c->n_acc = rank[j] + acc[j];
  }
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx != LLONG_MIN) atomicMax(&c->max_eid, mx);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x)
    keep[i] = acc[ev_edge(vals[i], directed)];
  if (blockIdx.x == 0 && threadIdx.x == 0) keep[E] = 0;
}

// pool-capacity check (block 0) + enumeration of the new blocks
__global__ void k_check_enumerate(const longlong4* __restrict__ off4, int64_t E, const IngestScalars* S, IngestCounters* c,
                                  const int64_t* __restrict__ ce_pend, const uint32_t* __restrict__ ce_ev, SegPlan P,
                                  const uint32_t* __restrict__ keys, const int64_t* __restrict__ seg_start,
                                  const int64_t* degree, int kind, int64_t tau, int64_t param, Recs R, longlong2* trig) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t ns = c->num_segs;  // off4 holds the scan up to num_segs (the total)
    c->new_blocks = off4[ns].x;
    c->new_slots = off4[ns].y;
    c->dir_need = off4[ns].z;
    if (c->new_slots > S->slots_free || c->dir_need > S->dir_free) c->abort |= ABORT_CAP;  // nothing written yet
  }
  const int64_t nseg = c->num_segs;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nb = P.nb_new[s];
    if (!nb) continue;
    const int64_t v = keys[seg_start[s]];
    const int64_t cs = P.cstart[s], cnt = P.acc_cnt[s], fill = P.fill[s];
    int64_t deg = degree[v] + fill, used = fill, rem = cnt - fill;
    int64_t r = off4[s].x;
    while (rem > 0) {
      const int64_t cap = sizing_cap(kind, tau, param, deg, ce_pend[cs + used]);
      const int64_t take = min(cap, rem);
      R.first[r] = used;
      R.count[r] = take;
      R.cap[r] = cap;
      R.seg[r] = (int32_t)s;
      R.key[r] = ce_ev[cs + used];
      trig[ce_ev[cs + used]] = make_longlong2(1, cap);  // allocation order = triggering event order
      r++;
      deg += take;
      used += take;
      rem -= take;
    }
  }
}

// One segment's commit (shared by k_commit and the cooperative path): its new blocks (handle and
// slot base from the allocation order), the directory, the node row and its NodeRec.
//   ev_ts(r): timestamp of the segment's r-th accepted event
//   blk(k):   NewBlk of the segment's k-th new block
struct NewBlk {
  int64_t h, base, first, count, cap;
};
template <class EvTs, class Blk>
__device__ __forceinline__ void commit_segment(int64_t v, int64_t cnt, int64_t t, int64_t fill, int64_t nb, int64_t dnew,
                                               int64_t dir_new_off, int64_t tail_size, EvTs ev_ts, Blk blk,
                                               const NodeArrays& N, const BlockArrays& B, const DirArrays& D, int kind) {
  const int64_t nb_old = N.num_blocks[v], ns_old = N.nslots[v], deg_old = N.degree[v], oo = N.dir_off[v];
  const int64_t doff = dnew > 0 ? dir_new_off : oo;
  const int64_t t_tmax = (t != GF_NO_BLOCK && fill > 0) ? ev_ts(fill - 1) : 0;
  // the node's directory moves to a larger region when it grows past its capacity
  if (nb > 0 && dnew > 0)
    for (int64_t w = 0; w < nb_old * DIRW; w++) D.e[doff * DIRW + w] = D.e[oo * DIRW + w];
  int64_t h_first = GF_NO_BLOCK, h_last = GF_NO_BLOCK, tmin_last = 0, tmax_last = 0, base_last = 0;
  int64_t h_prev = t;
  for (int64_t k = 0; k < nb; k++) {
    const NewBlk nbk = blk(k);
    const int64_t h = nbk.h;
    const int64_t tmin = ev_ts(nbk.first), tmax = ev_ts(nbk.first + nbk.count - 1);
    B.cap[h] = nbk.cap;
    B.size[h] = nbk.count;
    B.tmin[h] = tmin;
    B.tmax[h] = tmax;
    B.base[h] = nbk.base;
    B.prev[h] = h_prev;
    B.next[h] = GF_NO_BLOCK;
    if (k > 0) B.next[h_prev] = h;
    int64_t* e = D.e + (doff + nb_old + k) * DIRW;
    e[0] = tmin;
    e[1] = ns_old + nbk.first;
    e[2] = nbk.base;
    e[3] = tmax;
    if (k == 0) h_first = h;
    h_prev = h;
    h_last = h;
    tmin_last = tmin;
    tmax_last = tmax;
    base_last = nbk.base;
  }
  // a block allocated while live degree != slots written (a deletion happened) or by
  // batch sizing leaves the closed-form position -> block law (SizingLaw)
  if (nb > 0 && (kind == GF_SIZING_BATCH || deg_old != ns_old)) N.nflags[v] |= 1;
  int64_t tl_tmin = 0, tl_tmax = 0, tl_base = 0;
  if (t != GF_NO_BLOCK) {
    tl_tmin = B.tmin[t];
    tl_base = B.base[t];
    tl_tmax = fill > 0 ? t_tmax : B.tmax[t];
  }
  if (t != GF_NO_BLOCK && fill > 0) {
    B.size[t] = tail_size + fill;
    B.tmax[t] = t_tmax;
    D.e[(doff + nb_old - 1) * DIRW + 3] = t_tmax;  // old tail grew
  }
  if (nb > 0) {
    if (t == GF_NO_BLOCK) N.head[v] = h_first;
    else B.next[t] = h_first;
    tl_tmin = tmin_last;
    tl_tmax = tmax_last;
    tl_base = base_last;
    N.tail[v] = h_last;
    if (dnew > 0) {
      N.dir_off[v] = doff;
      N.dir_cap[v] = dnew;
    }
  }
  const int64_t nbt = nb_old + nb;
  N.num_blocks[v] = nbt;
  N.degree[v] = deg_old + cnt;
  N.nslots[v] = ns_old + cnt;
  int64_t* rr = N.nrec + v * NREC;
  rr[0] = doff;
  rr[1] = ns_old + cnt;
  rr[2] = nbt | (N.valid[v] ? NREC_VALID : 0) | ((N.nflags[v] & 1) ? NREC_IRREG : 0);
  rr[3] = D.e[doff * DIRW + 1];
  rr[4] = D.e[(doff + nbt - 1) * DIRW + 1];
  rr[5] = tl_base;
  rr[6] = tl_tmin;
  rr[7] = tl_tmax;
  rr[8] = D.e[doff * DIRW];
}

struct SlotArrays {
  Slot* slots;
  int64_t *sts, *fts;
  int32_t *sts32, *fts32;
  uint32_t* okbits;          // candidate bitmap, NULL before the first deletion
  const uint8_t* node_valid;
};

// one slot record plus its timestamp copies and fences
__device__ __forceinline__ void write_slot(const SlotArrays& SA, int64_t pos, int64_t ts, int64_t eid, int32_t nbr, int32_t owner) {
  Slot sl;
  sl.ts = ts;
  sl.eid = eid;
  sl.nbr = nbr;
  sl.owner = owner;
  sl.valid = 1;
  sl.pad = 0;
  SA.slots[pos] = sl;
  SA.sts[pos] = ts;
  if ((pos & (FENCE - 1)) == 0) SA.fts[pos / FENCE] = ts;
  const int32_t t32 = (int32_t)max(min(ts, (int64_t)INT32_MAX), (int64_t)INT32_MIN);  // exact while ts32
  SA.sts32[pos] = t32;
  if ((pos & (FENCE32 - 1)) == 0) SA.fts32[pos / FENCE32] = t32;
  if (SA.okbits) {  // a new edge is a candidate unless its neighbour was deleted
    const uint32_t bit = 1u << (pos & 31);
    if (SA.node_valid[nbr]) atomicOr(SA.okbits + (pos >> 5), bit);
    else atomicAnd(SA.okbits + (pos >> 5), ~bit);
  }
}

// The commit: one THREAD per segment writes its new blocks (handle and slot base from the trigger
// scan), the directory, the node and its NodeRec (a warp per segment serialised millions of
// segments per warp at 10M-edge batches); one thread per accepted event writes its slot.
// The capacity check ran in an earlier kernel, so a set abort flag is seen here.
__global__ void k_commit(const IngestCounters* c, const IngestScalars* S, const uint32_t* __restrict__ keys,
                         const int64_t* __restrict__ seg_start, SegPlan P, const longlong4* __restrict__ off4, Recs R,
                         const longlong2* __restrict__ tscan, const uint32_t* __restrict__ ce_ev,
                         const int64_t* __restrict__ rec, int directed, const int64_t* __restrict__ old_tail, NodeArrays N,
                         BlockArrays B, DirArrays D, int kind) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  const int64_t blk_used = S->blk_used, slots_used = S->slots_used, dir_used = S->dir_used, nfree = S->nfree;
  const int64_t* __restrict__ freel = S->free_list;
  // the r-th allocation of the batch takes free_handles.pop() while any are left, then a fresh handle
  auto handle_of = [&](int64_t r) { return r < nfree ? freel[nfree - 1 - r] : blk_used + (r - nfree); };
  const int64_t nseg = c->num_segs;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cnt = P.acc_cnt[s];
    if (!cnt) continue;
    const int64_t cs = P.cstart[s], r0 = off4[s].x;
    auto ev_ts = [&](int64_t r) { return rec[ER * ev_edge(ce_ev[cs + r], directed) + ER_TS]; };
    auto blk = [&](int64_t k) {
      const int64_t r = r0 + k;
      const longlong2 tr = tscan[R.key[r]];
      return NewBlk{handle_of(tr.x), slots_used + tr.y, R.first[r], R.count[r], R.cap[r]};
    };
    commit_segment(keys[seg_start[s]], cnt, old_tail[s], P.fill[s], P.nb_new[s], P.plan4[s].z, dir_used + off4[s].z,
                   P.tail_size[s], ev_ts, blk, N, B, D, kind);
  }
}

// slots: one thread per accepted event (a separate, register-light kernel: full occupancy for the
// latency-bound per-event chain)
__global__ void __launch_bounds__(256, 8)
    k_commit_slots(const IngestCounters* c, const IngestScalars* S, const uint32_t* __restrict__ keys,
                   const int64_t* __restrict__ seg_start, SegPlan P, const longlong4* __restrict__ off4, Recs R,
                   const longlong2* __restrict__ tscan, const uint32_t* __restrict__ ce_ev,
                   const int32_t* __restrict__ ce_seg, const int64_t* __restrict__ rec, int directed,
                   const int64_t* __restrict__ old_tail, const int64_t* __restrict__ bbase, SlotArrays SA) {
  pdl_enter();  // PDL: launched early by the previous kernel of the ingest graph
  if (c->abort) return;
  const int64_t slots_used = S->slots_used;
  const int64_t nseg = c->num_segs;
  const int64_t nacc_ev = P.cstart[nseg - 1] + P.acc_cnt[nseg - 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nacc_ev; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t sg = ce_seg[i];
    const int64_t r = i - P.cstart[sg];
    const uint32_t ev = ce_ev[i];
    const int64_t j = ev_edge(ev, directed);
    const int side = directed ? 0 : (int)(ev & 1);
    const int64_t fill = P.fill[sg];
    int64_t pos;
    if (r < fill) {
      pos = bbase[old_tail[sg]] + P.tail_size[sg] + r;  // the old tail's base does not change
    } else {
      int64_t lo = off4[sg].x, hi = lo + P.nb_new[sg];  // last rec with first <= r
      while (hi - lo > 1) {
        const int64_t m = (lo + hi) >> 1;
        if (R.first[m] <= r) lo = m;
        else hi = m;
      }
      pos = slots_used + tscan[R.key[lo]].y + (r - R.first[lo]);
    }
    const longlong4 er = reinterpret_cast<const longlong4*>(rec)[j];  // one sector
    write_slot(SA, pos, er.z, er.w, (int32_t)(side ? er.x : er.y), (int32_t)keys[seg_start[sg]]);
  }
}

// ---- cooperative single-launch ingest (the common case) ----------------------------
// One cooperative kernel replaces the ~20-node launch sequence when the batch can be planned
// without the rejection machinery (K1).  Its phases are separated by grid barriers:
//   A  stage the edge records; node / timestamp / id ranges; per-node event counts (persistent
//      zeroed counters; one atomic per node per 1024-event sub-chunk, aggregated in a shared-memory
//      hash) and the list of touched nodes, one segment each, in first-touch order
//   C  rows of new nodes; segment starts: a grid scan of the counts
//   D  events scattered into their segments (the same aggregation; the counters count back to 0)
//   E  each segment's events sorted by event index -- a warp bitonic sort up to 32 events, a rank
//      count up to 1024, a CTA radix sort up to CO_SORT -- so a segment lists its node's events in
//      append order
//   F  chronology check (any endpoint that could see a decreasing timestamp sends the batch to the
//      general sequence, storage.py:426-437); per-segment block plan (storage.py:449-459), which marks
//      the events that allocate, inside the reduce pass of its grid scan; then a grid scan over the
//      events in event order gives each new block its handle rank and slot base (the reference's
//      allocation order)
//   I  commit: blocks, directory, node rows, NodeRecs (a thread per segment), slots (a thread per
//      event; both walk the capacity law again instead of storing per-block records), edge ids
// Nothing is mutated before phase I except the rows of new nodes, which the general sequence
// initialises the same way, so every abort leaves the store as it was.
constexpr int CO_T = 1024;                  // threads per CTA
constexpr int CO_ITEMS = 8;                 // CTA radix sort: CO_T x CO_ITEMS keys
constexpr int CO_SORT = CO_T * CO_ITEMS;    // events per segment on this path
constexpr int CO_BITMAP_WORDS = 8 * CO_T;   // E-phase bitmap: batches of up to 2^18 events
constexpr int64_t CO_MAX_EVENTS = 1 << 22;


struct CoopBufs {
  uint32_t* sev;      // [E] event index per sorted position (segment-major, append order inside)
  int32_t* sseg;      // [E] segment of each sorted position
  int32_t* touched;   // [E] node of each segment
  int32_t* sstart;    // [E + 1] segment starts
  int32_t* big;       // [E] segments with more than 32 events
  int64_t* ctot;      // [grid * 8] per-CTA partial sums of the grid scans
  int64_t *fill, *tail_size, *old_tail, *nb_new, *deg0;  // [E] per segment
  int64_t *nb_old, *ns_old, *dir_old;                     // [E] per segment: node row before the batch
  int32_t* moves;                                         // [E] segments whose directory moves
  longlong4 *plan4, *off4;                                // [E + 1] per segment
  int64_t *trig, *trank, *tbase;  // [E] per event: capacity of the block it allocates (0: none), rank, slot base
  int32_t *ncnt, *nseg;           // per node (persistent)
};

template <class T>
__device__ __forceinline__ T ldl2(const T* p) { return __ldcg(p); }

__device__ __forceinline__ long long gtimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define COOP_MARK(i)                                            \
  do {                                                          \
    if (blockIdx.x == 0 && threadIdx.x == 0) c->phase_ns[i] = gtimer_ns(); \
  } while (0)  // data another CTA wrote in this launch

// exclusive scan of K int64 fields over the CTA (CO_T threads); returns the CTA total.  sm holds
// 33 rows: the 32 warp totals, scanned in place by warp 0, and the CTA total.
template <int K>
__device__ __forceinline__ void cta_scan(const int64_t (&x)[K], int64_t (&excl)[K], int64_t (&tot)[K], int64_t (*sm)[K]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t inc[K];
#pragma unroll
  for (int f = 0; f < K; f++) {
    int64_t v = x[f];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    inc[f] = v;
  }
  __syncthreads();  // sm may still be read by a previous call
  if (lane == 31)
#pragma unroll
    for (int f = 0; f < K; f++) sm[w][f] = inc[f];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int f = 0; f < K; f++) {
      const int64_t y = sm[lane][f];
      int64_t v = y;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t z = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += z;
      }
      sm[lane][f] = v - y;  // exclusive prefix of the warp totals
      if (lane == 31) sm[32][f] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int f = 0; f < K; f++) {
    excl[f] = sm[w][f] + inc[f] - x[f];
    tot[f] = sm[32][f];
  }
}

// Grid-wide exclusive scan (reduce, barrier, scan) of n items of K fields: val1(i, out[K]) gives
// item i in the reduce pass (it may compute and store it), val2 in the scan pass, put(i, excl[K])
// receives its exclusive prefix; gtot receives the total on every CTA.
template <int K, class V1, class V2, class O>
__device__ __forceinline__ void grid_scan(cg::grid_group& grid, int64_t n, V1 val1, V2 val2, O put, int64_t* ctot,
                                          int64_t (*sm)[K], int64_t (&gtot)[K]) {
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t chunk = ((n + G - 1) / G + CO_T - 1) / CO_T * CO_T;
  const int64_t lo = min(n, b * chunk), hi = min(n, lo + chunk);
  int64_t part[K], x1[K];  // x1: the item of a chunk of one round, kept for the scan pass
#pragma unroll
  for (int f = 0; f < K; f++) part[f] = x1[f] = 0;
  const bool one_round = hi - lo <= CO_T;
  for (int64_t i = lo + threadIdx.x; i < hi; i += CO_T) {
    int64_t x[K];
    val1(i, x);
#pragma unroll
    for (int f = 0; f < K; f++) {
      part[f] += x[f];
      x1[f] = x[f];
    }
  }
  int64_t ex[K], t[K];
  cta_scan<K>(part, ex, t, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int f = 0; f < K; f++) ctot[b * K + f] = t[f];
  grid.sync();
  // the CTA totals (G <= CO_T) are scanned by one CTA scan: thread i holds CTA i's total
  __shared__ int64_t s_base[K];
  int64_t base[K];
  {
    int64_t y[K];
#pragma unroll
    for (int f = 0; f < K; f++) y[f] = threadIdx.x < G ? ldl2(ctot + threadIdx.x * K + f) : 0;
    cta_scan<K>(y, ex, gtot, sm);
    if (threadIdx.x == b)
#pragma unroll
      for (int f = 0; f < K; f++) s_base[f] = ex[f];
    __syncthreads();
#pragma unroll
    for (int f = 0; f < K; f++) base[f] = s_base[f];
  }
  for (int64_t i0 = lo; i0 < hi; i0 += CO_T) {
    const int64_t i = i0 + threadIdx.x;
    int64_t x[K];
    if (i < hi && one_round)
#pragma unroll
      for (int f = 0; f < K; f++) x[f] = x1[f];
    else if (i < hi) val2(i, x);
    else
#pragma unroll
      for (int f = 0; f < K; f++) x[f] = 0;
    cta_scan<K>(x, ex, t, sm);
    if (i < hi) {
      int64_t o[K];
#pragma unroll
      for (int f = 0; f < K; f++) o[f] = base[f] + ex[f];
      put(i, o);
    }
#pragma unroll
    for (int f = 0; f < K; f++) base[f] += t[f];
  }
}

__device__ __forceinline__ int64_t ev_node(const int64_t* rec, uint32_t e, int directed) {
  const int64_t j = ev_edge(e, directed);
  return rec[ER * j + ((!directed && (e & 1)) ? ER_DST : ER_SRC)];
}

__global__ void __launch_bounds__(CO_T, 1)
    k_ingest_coop(const __grid_constant__ IngestScalars S_, IngestCounters* c, int64_t* rec, int64_t n, int directed,
                  int64_t node_cap, int sort_bits, CoopBufs CB, NodeArrays N, BlockArrays B, DirArrays D, SlotArrays SA,
                  int kind, int64_t tau, int64_t param, IngestCounters* hout) {
  // the per-call scalars arrive as a kernel parameter (no H2D copy ahead of the launch); the counters
  // go back the other way without a copy either: the last CTA to finish writes them to the pinned
  // host struct `hout` and re-arms `c` for the next call
  const IngestScalars* S = &S_;
  __shared__ long long s_abort;
  auto cta_abort = [&]() -> long long {  // c->abort as one value for the whole CTA
    __syncthreads();
    if (threadIdx.x == 0) s_abort = __ldcg(&c->abort);
    __syncthreads();
    return s_abort;
  };
  auto finish = [&]() {  // every CTA, on every exit
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd((unsigned long long*)&c->done, 1ull) == gridDim.x - 1) {
        __threadfence();
        const long long* w = reinterpret_cast<const long long*>(c);
        long long* o = reinterpret_cast<long long*>(hout);
        for (size_t i = 0; i < sizeof(IngestCounters) / sizeof(long long); i++) o[i] = __ldcg(w + i);
        counters_arm(c);
      }
    }
  };
  cg::grid_group grid = cg::this_grid();
  typedef cub::BlockRadixSort<uint32_t, CO_T, CO_ITEMS> BSortK;
  constexpr int HC = 2 * CO_T;  // per-CTA node hash: at most CO_T distinct nodes per sub-chunk
  __shared__ union {
    typename BSortK::TempStorage sortk;
    struct {
      int32_t key[HC], cnt[HC], base[HC], seg[HC];
    } h;
    uint32_t bits[CO_BITMAP_WORDS];  // E-phase rank bitmap over event indices
  } sm;
  __shared__ int64_t s_scan[CO_T / 32 + 1][4];
  __shared__ long long red[4][CO_T / 32];
  __shared__ uint32_t s_key[CO_T];
  const int64_t E = directed ? n : 2 * n;
  const int64_t gtid = blockIdx.x * (int64_t)CO_T + threadIdx.x, gstride = (int64_t)gridDim.x * CO_T;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool has_eids = S->eids_in != nullptr;
  // each CTA aggregates a contiguous chunk of events, CO_T at a time, in a shared-memory node hash
  const int64_t L = (E + gridDim.x - 1) / gridDim.x;
  const int64_t c_lo = min(E, (int64_t)blockIdx.x * L), c_hi = min(E, c_lo + L);
  auto node_in = [&](int64_t e) -> int64_t {
    const int64_t j = ev_edge((uint32_t)e, directed);
    return (!directed && (e & 1)) ? S->dst[j] : S->src[j];
  };
  auto h_clear = [&]() {
    for (int i = threadIdx.x; i < HC; i += CO_T) {
      sm.h.key[i] = -1;
      sm.h.cnt[i] = 0;
    }
  };
  auto h_insert = [&](int32_t v, int& slot) -> int {  // returns the event's rank among the sub-chunk's events of v
    unsigned hh = ((unsigned)v * 2654435761u) & (HC - 1);
    while (true) {
      const int k = atomicCAS(&sm.h.key[hh], -1, v);
      if (k == -1 || k == v) {
        slot = (int)hh;
        return atomicAdd(&sm.h.cnt[hh], 1);
      }
      hh = (hh + 1) & (HC - 1);
    }
  };

  COOP_MARK(0);
  // ---- A: stage; node / timestamp / id ranges; per-node counts, touched nodes ----
  {
    long long mn = LLONG_MAX, mx = LLONG_MIN, tn = LLONG_MAX, tx = LLONG_MIN, ex = LLONG_MIN;
    for (int64_t j = gtid; j < n; j += gstride) {
      const long long a = S->src[j], b = S->dst[j], t = S->ts[j], id = has_eids ? S->eids_in[j] : 0;
      reinterpret_cast<longlong4*>(rec)[j] = make_longlong4(a, b, t, id);
      mn = min(mn, min(a, b));
      mx = max(mx, max(a, b));
      tn = min(tn, t);
      tx = max(tx, t);
      ex = max(ex, id);
    }
    for (int64_t e = gtid; e < E; e += gstride) CB.trig[e] = 0;
    for (int o = 16; o; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      tn = min(tn, __shfl_xor_sync(0xffffffffu, tn, o));
      tx = max(tx, __shfl_xor_sync(0xffffffffu, tx, o));
      ex = max(ex, __shfl_xor_sync(0xffffffffu, ex, o));
    }
    if (lane == 0) {
      red[0][w] = mn;
      red[1][w] = mx;
      red[2][w] = tn;
      red[3][w] = tx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < CO_T / 32; i++) {
        mn = min(mn, red[0][i]);
        mx = max(mx, red[1][i]);
        tn = min(tn, red[2][i]);
        tx = max(tx, red[3][i]);
      }
      if (mn != LLONG_MAX) {
        atomicMin(&c->minv, mn);
        atomicMax(&c->maxv, mx);
        atomicMin(&c->tsmin, tn);
        atomicMax(&c->tsmax, tx);
      }
    }
    if (has_eids && lane == 0 && ex != LLONG_MIN) atomicMax(&c->max_eid, ex);
  }
  // a chunk of one sub-chunk (E <= grid x CO_T, the common case) keeps its hash in shared memory and
  // each event's slot and rank in registers for phase D, which then skips rebuilding the hash
  const bool one_sub = c_hi - c_lo <= CO_T;
  int a_slot = 0, a_lr = 0;
  for (int64_t s0 = c_lo; s0 < c_hi; s0 += CO_T) {
    __syncthreads();
    h_clear();
    __syncthreads();
    const int64_t e = s0 + threadIdx.x;
    if (e < c_hi) {
      const int64_t v = node_in(e);
      if (v < 0 || v >= node_cap) atomicOr((unsigned long long*)&c->abort, (unsigned long long)ABORT_NODES);
      else a_lr = h_insert((int32_t)v, a_slot);
    }
    __syncthreads();
    // one counter atomic per (sub-chunk, node); the first to count a node lists it (one segment)
#ifndef GF_AB_SEG_WARP
    {  // the sub-chunk's fresh nodes take one range of the segment list: one list atomic per CTA
      int32_t kk[HC / CO_T];
      bool fr[HC / CO_T];
      int64_t nf[1] = {0}, ex[1], tt[1];
#pragma unroll
      for (int q = 0; q < HC / CO_T; q++) {
        const int i = q * CO_T + threadIdx.x;
        kk[q] = sm.h.key[i];
        fr[q] = kk[q] >= 0 && atomicAdd(&CB.ncnt[kk[q]], sm.h.cnt[i]) == 0;
        nf[0] += fr[q] ? 1 : 0;
      }
      cta_scan<1>(nf, ex, tt, reinterpret_cast<int64_t(*)[1]>(s_scan));
      __shared__ unsigned long long s_segbase;
      if (threadIdx.x == 0) s_segbase = tt[0] ? atomicAdd((unsigned long long*)&c->num_segs, (unsigned long long)tt[0]) : 0ull;
      __syncthreads();
      int64_t pos = (int64_t)s_segbase + ex[0];
#pragma unroll
      for (int q = 0; q < HC / CO_T; q++)
        if (fr[q]) CB.touched[pos++] = kk[q];
    }
#else
    for (int i0 = 0; i0 < HC; i0 += CO_T) {
      const int i = i0 + threadIdx.x;
      const int32_t k = sm.h.key[i];
      const bool fresh = k >= 0 && atomicAdd(&CB.ncnt[k], sm.h.cnt[i]) == 0;
      const unsigned fm = __ballot_sync(0xffffffffu, fresh);
      unsigned long long base = 0;
      if (fm && lane == __ffs(fm) - 1) base = atomicAdd((unsigned long long*)&c->num_segs, (unsigned long long)__popc(fm));
      base = __shfl_sync(0xffffffffu, base, fm ? __ffs(fm) - 1 : 0);
      if (fresh) CB.touched[base + __popc(fm & ((1u << lane) - 1))] = k;
    }
#endif
  }
  grid.sync();

  COOP_MARK(1);
  const int64_t nseg = ldl2(&c->num_segs);
  if (cta_abort() & ABORT_NODES) {  // node ids beyond the table (or negative): undo the counts
    for (int64_t i = gtid; i < nseg; i += gstride) CB.ncnt[ldl2(&CB.touched[i])] = 0;
    finish();
    return;
  }
  // ---- C: rows of new nodes; segment starts ----
  const long long maxv = ldl2(&c->maxv);
  for (int64_t v = S->num_nodes + gtid; v < maxv + 1; v += gstride) {
    N.head[v] = GF_NO_BLOCK;
    N.tail[v] = GF_NO_BLOCK;
    N.num_blocks[v] = 0;
    N.degree[v] = 0;
    const_cast<uint8_t*>(N.valid)[v] = 1;
    N.nslots[v] = 0;
    N.dir_off[v] = -1;
    N.dir_cap[v] = 0;
    N.nflags[v] = 0;
    int64_t* r = N.nrec + v * NREC;
    r[0] = -1;
    r[1] = 0;
    r[2] = NREC_VALID;
    for (int k = 3; k < NREC; k++) r[k] = 0;
  }
  {
    auto cnt_of = [&](int64_t i, int64_t (&x)[1]) { x[0] = ldl2(&CB.ncnt[ldl2(&CB.touched[i])]); };
    int64_t tot[1];
    grid_scan<1>(
        grid, nseg, cnt_of, cnt_of,
        [&](int64_t i, int64_t (&o)[1]) {
          const int32_t v = ldl2(&CB.touched[i]);
          const int64_t m = ldl2(&CB.ncnt[v]);
          CB.sstart[i] = (int32_t)o[0];
          CB.nseg[v] = (int32_t)i;
          if (m > 32) {
            CB.big[atomicAdd((unsigned long long*)&c->num_big, 1ull)] = (int32_t)i;
            if (m > CO_SORT) atomicOr((unsigned long long*)&c->abort, (unsigned long long)ABORT_SLOW);
          }
        },
        CB.ctot, reinterpret_cast<int64_t(*)[1]>(s_scan), tot);
    if (gtid == 0) CB.sstart[nseg] = (int32_t)E;
  }
  grid.sync();

  COOP_MARK(2);
  // ---- D: scatter, one counter atomic per (sub-chunk, node); the counters count back to zero ----
  for (int64_t s0 = c_lo; s0 < c_hi; s0 += CO_T) {
    const int64_t e = s0 + threadIdx.x;
    int slot = a_slot, lr = a_lr;
#ifndef GF_AB_NO_HASH_REUSE
    if (!one_sub)
#endif
    {
      __syncthreads();
      h_clear();
      __syncthreads();
      if (e < c_hi) lr = h_insert((int32_t)node_in(e), slot);
      __syncthreads();
    }
    for (int i = threadIdx.x; i < HC; i += CO_T) {
      const int32_t k = sm.h.key[i];
      if (k >= 0) {
        const int m = sm.h.cnt[i];
        const int top = atomicSub(&CB.ncnt[k], m);  // this sub-chunk takes [top - m, top) of the segment
        const int32_t sg = ldl2(&CB.nseg[k]);
        sm.h.base[i] = ldl2(&CB.sstart[sg]) + top - m;
        sm.h.seg[i] = sg;
      }
    }
    __syncthreads();
    if (e < c_hi) {
      const int64_t p = sm.h.base[slot] + lr;
      CB.sev[p] = (uint32_t)e;
      CB.sseg[p] = sm.h.seg[slot];
    }
  }
  grid.sync();
  if (cta_abort()) {  // a segment beyond one CTA's sort
    finish();
    return;
  }

  COOP_MARK(3);
  // ---- E: each segment in append order ----
  {
    const int64_t gw = gtid >> 5, nw = gstride >> 5;
    for (int64_t sg = gw; sg < nseg; sg += nw) {
      const int32_t st = ldl2(&CB.sstart[sg]), m = ldl2(&CB.sstart[sg + 1]) - st;
      if (m < 2 || m > 32) continue;
      uint32_t x = lane < m ? ldl2(&CB.sev[st + lane]) : 0xffffffffu;
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
          x = (((lane & j) == 0) == ((lane & k) == 0)) ? min(x, y) : max(x, y);
        }
      if (lane < m) CB.sev[st + lane] = x;
    }
    __syncthreads();
    COOP_MARK(7);
    const int64_t nbig = ldl2(&c->num_big);
    for (int64_t bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
      const int32_t sg = ldl2(&CB.big[bi]);
      const int32_t st = ldl2(&CB.sstart[sg]), m = ldl2(&CB.sstart[sg + 1]) - st;
      if (m <= 256) {
        // event indices are distinct: a key's rank is the number of smaller keys in the segment
        const uint32_t x = threadIdx.x < m ? ldl2(&CB.sev[st + threadIdx.x]) : 0u;
        __syncthreads();
        if (threadIdx.x < m) s_key[threadIdx.x] = x;
        __syncthreads();
        if (threadIdx.x < m) {
          int rank = 0;
          for (int i = 0; i < m; i++) rank += s_key[i] < x ? 1 : 0;
          CB.sev[st + rank] = x;
        }
        continue;
      }
      if (E <= 32 * CO_BITMAP_WORDS) {
        // a bitmap over [0, E): a key's rank is the number of set bits below it (thread t owns words
        // 8t .. 8t+7 and their prefix count in s_key[t])
        const int nw = (int)((E + 31) >> 5);
        uint32_t keys[CO_ITEMS];
#pragma unroll
        for (int k = 0; k < CO_ITEMS; k++) {
          const int i = k * CO_T + threadIdx.x;
          keys[k] = i < m ? ldl2(&CB.sev[st + i]) : 0xffffffffu;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nw; i += CO_T) sm.bits[i] = 0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < CO_ITEMS; k++)
          if (keys[k] != 0xffffffffu) atomicOr(&sm.bits[keys[k] >> 5], 1u << (keys[k] & 31));
        __syncthreads();
        int64_t cnt8[1] = {0};
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const int wi = threadIdx.x * 8 + q;
          cnt8[0] += wi < nw ? __popc(sm.bits[wi]) : 0;
        }
        int64_t ex1[1], tt1[1];
        cta_scan<1>(cnt8, ex1, tt1, reinterpret_cast<int64_t(*)[1]>(s_scan));
        s_key[threadIdx.x] = (uint32_t)ex1[0];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < CO_ITEMS; k++) {
          const uint32_t x = keys[k];
          if (x == 0xffffffffu) continue;
          const int wi = (int)(x >> 5), g0 = wi & ~7;
          int rank = (int)s_key[wi >> 3] + __popc(sm.bits[wi] & ((1u << (x & 31)) - 1));
          for (int q = g0; q < wi; q++) rank += __popc(sm.bits[q]);
          CB.sev[st + rank] = x;
        }
        __syncthreads();
        continue;
      }
      uint32_t keys[CO_ITEMS];
#pragma unroll
      for (int k = 0; k < CO_ITEMS; k++) {
        const int i = threadIdx.x * CO_ITEMS + k;
        keys[k] = i < m ? ldl2(&CB.sev[st + i]) : 0xffffffffu;
      }
      __syncthreads();
      BSortK(sm.sortk).Sort(keys, 0, sort_bits);
#pragma unroll
      for (int k = 0; k < CO_ITEMS; k++) {
        const int i = threadIdx.x * CO_ITEMS + k;
        if (i < m) CB.sev[st + i] = keys[k];
      }
    }
  }
  grid.sync();

  COOP_MARK(4);
  // ---- F: chronology; per-segment block plan, its allocation triggers and its scan ----
  for (int64_t p = gtid; p < E; p += gstride) {
    const int32_t sg = ldl2(&CB.sseg[p]);
    const uint32_t e = ldl2(&CB.sev[p]);
    const int64_t t = rec[ER * ev_edge(e, directed) + ER_TS];
    bool viol;
    if (p == ldl2(&CB.sstart[sg])) viol = t < node_tmax(N.tail, B.size, B.tmax, ev_node(rec, e, directed));
    else viol = t < rec[ER * ev_edge(ldl2(&CB.sev[p - 1]), directed) + ER_TS];
    if (viol) atomicOr((unsigned long long*)&c->abort, (unsigned long long)ABORT_SLOW);
  }
  __syncthreads();
  COOP_MARK(8);
  int64_t tot3[3];
  grid_scan<3>(
      grid, nseg,
      [&](int64_t sg, int64_t (&x)[3]) {  // pass 1: the plan (storage.py:449-459 capacity law per allocation)
        const int64_t v = ldl2(&CB.touched[sg]);
        const int64_t st = ldl2(&CB.sstart[sg]), cnt = ldl2(&CB.sstart[sg + 1]) - st;
        const int64_t t = ldl2(&N.tail[v]), deg0 = ldl2(&N.degree[v]);
        int64_t fill = 0, tsz = 0;
        if (t != GF_NO_BLOCK) {
          tsz = B.size[t];
          fill = min(B.cap[t] - tsz, cnt);
        }
        CB.old_tail[sg] = t;
        CB.fill[sg] = fill;
        CB.tail_size[sg] = tsz;
        CB.deg0[sg] = deg0;
        int64_t deg = deg0 + fill, used = fill, blocks = 0, slots = 0;
        while (used < cnt) {
          const int64_t cap = sizing_cap(kind, tau, param, deg, cnt - used);  // pending: no rejections here
          const int64_t take = min(cap, cnt - used);
          CB.trig[ldl2(&CB.sev[st + used])] = cap;  // the event that allocates this block
          blocks++;
          slots += cap;
          deg += take;
          used += take;
        }
        CB.nb_new[sg] = blocks;
        const int64_t nbo = ldl2(&N.num_blocks[v]), need = nbo + blocks;
        CB.nb_old[sg] = nbo;
        CB.ns_old[sg] = ldl2(&N.nslots[v]);
        CB.dir_old[sg] = ldl2(&N.dir_off[v]);
        int64_t dnew = 0;
        if (need > ldl2(&N.dir_cap[v])) {
          dnew = 8;
          while (dnew < need) dnew <<= 1;
          if (nbo > 0) CB.moves[atomicAdd((unsigned long long*)&c->num_moves, 1ull)] = (int32_t)sg;
        }
        CB.plan4[sg] = make_longlong4(blocks, slots, dnew, 0);
        x[0] = blocks;
        x[1] = slots;
        x[2] = dnew;
      },
      [&](int64_t sg, int64_t (&x)[3]) {  // pass 2: the stored plan
        x[0] = ldl2(&CB.plan4[sg].x);
        x[1] = ldl2(&CB.plan4[sg].y);
        x[2] = ldl2(&CB.plan4[sg].z);
      },
      [&](int64_t i, int64_t (&o)[3]) { CB.off4[i] = make_longlong4(o[0], o[1], o[2], 0); },
      CB.ctot, reinterpret_cast<int64_t(*)[3]>(s_scan), tot3);
  COOP_MARK(9);
  // abort is read once per CTA: CTA 0 may set ABORT_CAP below while another CTA (or a lagging warp)
  // is still at this check, and every thread of a CTA must leave through the same finish()
  if (cta_abort()) {  // a possible rejection: the general sequence resolves the batch
    finish();
    return;
  }
  if (tot3[1] > S->slots_free || tot3[2] > S->dir_free || tot3[0] - S->nfree > S->blocks_free) {
    if (gtid == 0) {
      c->new_blocks = tot3[0];
      c->new_slots = tot3[1];
      c->dir_need = tot3[2];
      c->abort |= ABORT_CAP;
    }
    finish();
    return;  // every CTA holds the same totals
  }
  if (gtid == 0) {
    c->new_blocks = tot3[0];
    c->new_slots = tot3[1];
    c->dir_need = tot3[2];
    c->n_acc = n;
  }
  {
    // handle rank and slot base of each new block: a scan of (1, capacity) over the triggering
    // events in event order = the reference's allocation order
    auto trig_of = [&](int64_t e, int64_t (&x)[2]) {
      const int64_t cap = ldl2(&CB.trig[e]);
      x[0] = cap > 0 ? 1 : 0;
      x[1] = cap;
    };
    int64_t tot2[2];
    grid_scan<2>(
        grid, E, trig_of, trig_of,
        [&](int64_t e, int64_t (&o)[2]) {
          if (ldl2(&CB.trig[e]) > 0) {
            CB.trank[e] = o[0];
            CB.tbase[e] = o[1];
          }
        },
        CB.ctot + 4 * gridDim.x, reinterpret_cast<int64_t(*)[2]>(s_scan), tot2);
  }
  __syncthreads();
  COOP_MARK(10);
  grid.sync();

  COOP_MARK(5);
  // ---- I: commit ----
  // Work is spread so that no thread walks a long serial chain: a directory that moves is copied by
  // one whole CTA; each new block is written by the thread of its allocating event; a segment's own
  // thread writes only the node row, the old tail and the NodeRec (storage.py:449-477).
  const int64_t blk_used = S->blk_used, slots_used = S->slots_used, dir_used = S->dir_used, nfree = S->nfree;
  const int64_t* __restrict__ freel = S->free_list;
  auto handle_of = [&](int64_t r) { return r < nfree ? freel[nfree - 1 - r] : blk_used + (r - nfree); };
  auto ts_of = [&](uint32_t e) { return rec[ER * ev_edge(e, directed) + ER_TS]; };
  const int64_t next_id = S->next_edge_id;
  const int64_t nmov = ldl2(&c->num_moves);
  for (int64_t mi = blockIdx.x; mi < nmov; mi += gridDim.x) {
    const int32_t sg = ldl2(&CB.moves[mi]);
    const int64_t from = ldl2(&CB.dir_old[sg]) * DIRW, to = (dir_used + ldl2(&CB.off4[sg].z)) * DIRW;
    const int64_t words = ldl2(&CB.nb_old[sg]) * DIRW, fill = ldl2(&CB.fill[sg]);
    // the old tail's tmax (its entry's last word) grows when the batch fills the tail
    const int64_t t_tmax = fill > 0 ? ts_of(ldl2(&CB.sev[ldl2(&CB.sstart[sg]) + fill - 1])) : 0;
    for (int64_t wd = threadIdx.x; wd < words; wd += CO_T) D.e[to + wd] = (fill > 0 && wd == words - 1) ? t_tmax : D.e[from + wd];
  }
  for (int64_t idx = gtid; idx < nseg + E; idx += gstride) {
    if (idx < nseg) {
      const int64_t sg = idx;
      const int64_t v = ldl2(&CB.touched[sg]);
      const int64_t st = ldl2(&CB.sstart[sg]), cnt = ldl2(&CB.sstart[sg + 1]) - st;
      const int64_t fill = ldl2(&CB.fill[sg]), deg0 = ldl2(&CB.deg0[sg]), nb = ldl2(&CB.nb_new[sg]);
      const int64_t dnew = ldl2(&CB.plan4[sg].z), t = ldl2(&CB.old_tail[sg]), tsz = ldl2(&CB.tail_size[sg]);
      const int64_t nb_old = ldl2(&CB.nb_old[sg]), ns_old = ldl2(&CB.ns_old[sg]), oo = ldl2(&CB.dir_old[sg]);
      const int64_t doff = dnew > 0 ? dir_used + ldl2(&CB.off4[sg].z) : oo;
      const int64_t t_tmax = (t != GF_NO_BLOCK && fill > 0) ? ts_of(ldl2(&CB.sev[st + fill - 1])) : 0;
      int64_t used = fill, deg = deg0 + fill, used_last = fill;
      for (int64_t k = 0; k < nb; k++) {  // the capacity law again: first rank of the last new block
        const int64_t cap = sizing_cap(kind, tau, param, deg, cnt - used), take = min(cap, cnt - used);
        used_last = used;
        used += take;
        deg += take;
      }
      int64_t tl_tmin = 0, tl_tmax = 0, tl_base = 0;
      if (t != GF_NO_BLOCK) {
        tl_tmin = B.tmin[t];
        tl_base = B.base[t];
        tl_tmax = fill > 0 ? t_tmax : B.tmax[t];
      }
      if (t != GF_NO_BLOCK && fill > 0) {
        B.size[t] = tsz + fill;
        B.tmax[t] = t_tmax;
        if (dnew == 0) D.e[(oo + nb_old - 1) * DIRW + 3] = t_tmax;  // a moving directory's copy carries it
      }
      uint8_t fl = N.nflags[v];
      if (nb > 0) {
        const uint32_t ef = ldl2(&CB.sev[st + fill]), el = ldl2(&CB.sev[st + used_last]);
        const int64_t h_first = handle_of(ldl2(&CB.trank[ef])), h_last = handle_of(ldl2(&CB.trank[el]));
        if (t == GF_NO_BLOCK) N.head[v] = h_first;
        else B.next[t] = h_first;
        N.tail[v] = h_last;
        tl_tmin = ts_of(el);
        tl_tmax = ts_of(ldl2(&CB.sev[st + cnt - 1]));
        tl_base = slots_used + ldl2(&CB.tbase[el]);
        if (dnew > 0) {
          N.dir_off[v] = doff;
          N.dir_cap[v] = dnew;
        }
        // a block allocated while live degree != slots written (a deletion happened) or by batch
        // sizing leaves the closed-form position -> block law (SizingLaw)
        if (kind == GF_SIZING_BATCH || deg0 != ns_old) {
          fl |= 1;
          N.nflags[v] = fl;
        }
      }
      const int64_t nbt = nb_old + nb;
      N.num_blocks[v] = nbt;
      N.degree[v] = deg0 + cnt;
      N.nslots[v] = ns_old + cnt;
      int64_t* rr = N.nrec + v * NREC;
      rr[0] = doff;
      rr[1] = ns_old + cnt;
      rr[2] = nbt | (N.valid[v] ? NREC_VALID : 0) | ((fl & 1) ? NREC_IRREG : 0);
      rr[3] = nb_old > 0 ? D.e[oo * DIRW + 1] : ns_old;  // entries of the old location: never rewritten
      rr[4] = nb > 0 ? ns_old + used_last : D.e[(oo + nb_old - 1) * DIRW + 1];
      rr[5] = tl_base;
      rr[6] = tl_tmin;
      rr[7] = tl_tmax;
      rr[8] = nb_old > 0 ? D.e[oo * DIRW] : ts_of(ldl2(&CB.sev[st]));
    } else {
      const int64_t p = idx - nseg;
      const int32_t sg = ldl2(&CB.sseg[p]);
      const int64_t st = ldl2(&CB.sstart[sg]), cnt = ldl2(&CB.sstart[sg + 1]) - st, r = p - st;
      const uint32_t e = ldl2(&CB.sev[p]);
      const int64_t j = ev_edge(e, directed), fill = ldl2(&CB.fill[sg]);
      const longlong4 er = reinterpret_cast<const longlong4*>(rec)[j];
      int64_t pos;
      if (r < fill) {
        pos = B.base[ldl2(&CB.old_tail[sg])] + ldl2(&CB.tail_size[sg]) + r;  // the old tail's base does not change
      } else {  // walk the segment's new blocks (the capacity law again) to the one holding rank r
        int64_t used = fill, deg = ldl2(&CB.deg0[sg]) + fill, prev_used = -1, k = 0;
        while (true) {
          const int64_t cap = sizing_cap(kind, tau, param, deg, cnt - used);
          const int64_t take = min(cap, cnt - used);
          if (r < used + take) {
            const uint32_t et = (r == used) ? e : ldl2(&CB.sev[st + used]);  // the block's allocating event
            const int64_t base = slots_used + ldl2(&CB.tbase[et]);
            pos = base + (r - used);
            if (r == used) {  // this event allocates block k of the segment: write it
              const int64_t h = handle_of(ldl2(&CB.trank[e]));
              const int64_t nbk = ldl2(&CB.nb_new[sg]), dnew = ldl2(&CB.plan4[sg].z);
              const int64_t doff = dnew > 0 ? dir_used + ldl2(&CB.off4[sg].z) : ldl2(&CB.dir_old[sg]);
              const int64_t tmax = ts_of(ldl2(&CB.sev[st + used + take - 1]));
              const int64_t prev = k == 0 ? ldl2(&CB.old_tail[sg]) : handle_of(ldl2(&CB.trank[ldl2(&CB.sev[st + prev_used])]));
              const int64_t next = k == nbk - 1 ? GF_NO_BLOCK : handle_of(ldl2(&CB.trank[ldl2(&CB.sev[st + used + take])]));
              B.cap[h] = cap;
              B.size[h] = take;
              B.tmin[h] = er.z;
              B.tmax[h] = tmax;
              B.base[h] = base;
              B.prev[h] = prev;
              B.next[h] = next;
              int64_t* de = D.e + (doff + ldl2(&CB.nb_old[sg]) + k) * DIRW;
              de[0] = er.z;
              de[1] = ldl2(&CB.ns_old[sg]) + used;
              de[2] = base;
              de[3] = tmax;
            }
            break;
          }
          prev_used = used;
          used += take;
          deg += take;
          k++;
        }
      }
      const int side = directed ? 0 : (int)(e & 1);
      write_slot(SA, pos, er.z, has_eids ? er.w : next_id + j, (int32_t)(side ? er.x : er.y),
                 (int32_t)(side ? er.y : er.x));
    }
  }
  for (int64_t j = gtid; j < n; j += gstride) S->out_eids[j] = has_eids ? rec[ER * j + ER_EID] : next_id + j;
  __syncthreads();
  COOP_MARK(6);
  finish();
}

// node capacity only (rows are initialised on the device by k_grow_nodes)
gf_status grow_node_cap(gf_graph* g, int64_t need, cudaStream_t s) {
  if (need <= g->node_cap) return GF_OK;
  g->gen++;
  int64_t nc = std::max<int64_t>(need, std::max<int64_t>(1024, g->node_cap * 2));
  int64_t k = g->num_nodes;
  GF_TRY(grow_array(g->head, k, nc, s));
  GF_TRY(grow_array(g->tail, k, nc, s));
  GF_TRY(grow_array(g->num_blocks, k, nc, s));
  GF_TRY(grow_array(g->degree, k, nc, s));
  GF_TRY(grow_array(g->node_valid, k, nc, s));
  GF_TRY(grow_array(g->nslots, k, nc, s));
  GF_TRY(grow_array(g->dir_off, k, nc, s));
  GF_TRY(grow_array(g->dir_cap, k, nc, s));
  GF_TRY(grow_array(g->nflags, k, nc, s));
  GF_TRY(grow_array(g->nrec, k * NREC, nc * NREC, s));
  g->node_cap = nc;
  return GF_OK;
}

// Host state after a committed batch (both paths): cursors, id counter, node count, 32-bit fences.
void apply_ingest(gf_graph* g, const IngestCounters& hc, int64_t nfree, bool user_eids, int64_t n, int64_t* h_rej) {
  if (hc.maxv + 1 > g->num_nodes) g->num_nodes = hc.maxv + 1;  // storage.py:410-412
  const int64_t nrec = hc.new_blocks;
  g->blk_used += std::max<int64_t>(0, nrec - nfree);  // fresh handles only
  g->free_handles.resize(nfree - std::min(nfree, nrec));
  g->slots_used += hc.new_slots;
  g->dir_used += hc.dir_need;
  if (user_eids) {
    if (hc.n_acc > 0 && hc.max_eid + 1 > g->next_edge_id) g->next_edge_id = hc.max_eid + 1;
  } else {
    g->next_edge_id += hc.n_acc;
  }
  g->total_edges_inserted += hc.n_acc;
  if (hc.tsmin < INT32_MIN || hc.tsmax > INT32_MAX) g->ts32 = 0;  // the 32-bit fence is no longer exact
  if (h_rej) *h_rej = n - hc.n_acc;
}

// handles freed by offload, copied for the commit (read on the device)
gf_status stage_free_handles(gf_graph* g, cudaStream_t s) {
  const int64_t nfree = (int64_t)g->free_handles.size();
  if (nfree > g->free_dev_cap) {
    if (g->free_dev) GF_CUDA(cudaFreeAsync(g->free_dev, s));
    g->free_dev = nullptr;
    g->free_dev_cap = 0;
    GF_CUDA(cudaMallocAsync(&g->free_dev, sizeof(int64_t) * (size_t)(2 * nfree), s));
    g->free_dev_cap = 2 * nfree;
  }
  if (nfree) GF_CUDA(cudaMemcpyAsync(g->free_dev, g->free_handles.data(), sizeof(int64_t) * nfree, cudaMemcpyHostToDevice, s));
  return GF_OK;
}

bool coop_enabled() {
  const char* e = getenv("GF_INGEST_NO_COOP");  // A/B and tests: force the general launch sequence
  return !(e && *e && *e != '0');
}

int coop_occupancy() {
  static int occ = -1;
  if (occ < 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ingest_coop, CO_T, 0) != cudaSuccess) occ = 0;
    cudaGetLastError();
  }
  return occ;
}

// scratch of the cooperative path for a batch of n edges on `grid` CTAs
std::tuple<IngestScalars*, IngestCounters*, int64_t*> coop_layout(Arena& a, const gf_graph* g, int64_t n, int64_t grid,
                                                                  CoopBufs& CB) {
  const int64_t E = g->directed ? n : 2 * n;
  void* p0 = a.take<IngestScalars>(1);
  void* p1 = a.take<IngestCounters>(1);
  void* p2 = a.take<longlong4>(n);
  CB.sev = a.take<uint32_t>(E);
  CB.sseg = a.take<int32_t>(E);
  CB.touched = a.take<int32_t>(E);
  CB.sstart = a.take<int32_t>(E + 1);
  CB.big = a.take<int32_t>(E);
  CB.ctot = a.take<int64_t>(grid * 8);
  CB.fill = a.take<int64_t>(E);
  CB.tail_size = a.take<int64_t>(E);
  CB.old_tail = a.take<int64_t>(E);
  CB.nb_new = a.take<int64_t>(E);
  CB.deg0 = a.take<int64_t>(E);
  CB.nb_old = a.take<int64_t>(E);
  CB.ns_old = a.take<int64_t>(E);
  CB.dir_old = a.take<int64_t>(E);
  CB.moves = a.take<int32_t>(E);
  CB.plan4 = a.take<longlong4>(E + 1);
  CB.off4 = a.take<longlong4>(E + 1);
  CB.trig = a.take<int64_t>(E);
  CB.trank = a.take<int64_t>(E);
  CB.tbase = a.take<int64_t>(E);
  CB.ncnt = g->co_ncnt;
  CB.nseg = g->co_nseg;
  return std::make_tuple((IngestScalars*)p0, (IngestCounters*)p1, (int64_t*)p2);
}

// per-node counters (zero between batches) and segment indices for the node table's capacity;
// scratch for a batch of n edges
gf_status ensure_coop(gf_graph* g, int64_t n, int64_t grid, cudaStream_t s) {
  if (g->co_node_cap < g->node_cap) {
    if (g->co_ncnt) GF_CUDA(cudaFreeAsync(g->co_ncnt, s));
    if (g->co_nseg) GF_CUDA(cudaFreeAsync(g->co_nseg, s));
    g->co_ncnt = g->co_nseg = nullptr;
    g->co_node_cap = 0;
    GF_CUDA(cudaMallocAsync(&g->co_ncnt, sizeof(int32_t) * (size_t)g->node_cap, s));
    GF_CUDA(cudaMallocAsync(&g->co_nseg, sizeof(int32_t) * (size_t)g->node_cap, s));
    GF_CUDA(cudaMemsetAsync(g->co_ncnt, 0, sizeof(int32_t) * (size_t)g->node_cap, s));
    g->co_node_cap = g->node_cap;
  }
  Arena probe;
  CoopBufs CB;
  coop_layout(probe, g, n, grid, CB);
  if (probe.off + 4096 > g->co_bytes) {
    if (g->co_buf) GF_CUDA(cudaFreeAsync(g->co_buf, s));
    g->co_buf = nullptr;
    g->co_bytes = 0;
    const size_t want = probe.off + 4096 + (probe.off + 4096) / 4;
    GF_CUDA(cudaMallocAsync(&g->co_buf, want, s));
    g->co_bytes = want;
    // the counters sit at a fixed offset of the buffer; armed once here, then by every launch's last CTA
    Arena A;
    A.base = (char*)g->co_buf;
    IngestCounters* dc = std::get<1>(coop_layout(A, g, n, grid, CB));
    IngestCounters armed;
    counters_arm(&armed);
    GF_CUDA(cudaMemcpyAsync(dc, &armed, sizeof(armed), cudaMemcpyHostToDevice, s));  // pageable: staged before return
  }
  return GF_OK;
}

// The cooperative single-launch path.  *done = false sends the batch to add_edges_fast (ABORT_SLOW,
// oversized batch, or no co-resident grid); nothing was mutated in that case.
gf_status add_edges_coop(gf_graph* g, const int64_t* src_in, const int64_t* dst_in, const int64_t* ts_in, int64_t n,
                         const int64_t* eids_user, int64_t* out_user, int64_t* h_rej, cudaStream_t s, bool* done) {
  *done = false;
  const int dir = g->directed;
  const int64_t E = dir ? n : 2 * n;
  if (E > CO_MAX_EVENTS || !coop_enabled()) return GF_OK;
  const int occ = coop_occupancy();
  if (occ < 1) return GF_OK;
  // enough threads for one segment or event each in the commit phase (segments <= events)
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms() * occ, (2 * E + CO_T - 1) / CO_T));
  if (g->node_cap == 0) GF_TRY(grow_node_cap(g, 1024, s));
  if (!g->ing_host) GF_CUDA(cudaMallocHost(&g->ing_host, 4096));
  GF_TRY(stage_free_handles(g, s));
  const int64_t nfree = (int64_t)g->free_handles.size();
  IngestScalars* hs = (IngestScalars*)g->ing_host;
  IngestCounters* hcp = (IngestCounters*)((char*)g->ing_host + 2048);
  IngestCounters hc;
  for (int attempt = 0;; attempt++) {
    GF_TRY(ensure_coop(g, n, grid, s));
    CoopBufs CB;
    Arena A;
    A.base = (char*)g->co_buf;
    auto [ds, dc, rec] = coop_layout(A, g, n, grid, CB);
    *hs = IngestScalars{src_in, dst_in, ts_in, eids_user, out_user, g->num_nodes, g->blk_used, g->slots_used,
                        g->dir_used, g->next_edge_id, g->slot_cap - g->slots_used, g->dir_cap_total - g->dir_used,
                        g->free_dev, nfree, g->blk_cap - g->blk_used};
    (void)ds;
    NodeArrays N{g->head, g->tail, g->num_blocks, g->degree, g->nslots, g->dir_off, g->dir_cap, g->node_valid,
                 g->nflags, g->nrec};
    BlockArrays B{g->bcap, g->bsize, g->btmin, g->btmax, g->bprev, g->bnext, g->bbase};
    DirArrays D{g->dir};
    SlotArrays SA{g->slots, g->sts, g->fts, g->sts32, g->fts32, g->okbits, g->node_valid};
    const IngestScalars a_S = *hs;
    int64_t a_n = n, a_cap = g->node_cap, a_tau = g->tau, a_param = g->sizing_param;
    int a_dir = dir, a_bits = bits_for(E + 1), a_kind = g->sizing_kind;
    void* args[] = {(void*)&a_S, (void*)&dc, (void*)&rec, (void*)&a_n, (void*)&a_dir, (void*)&a_cap, (void*)&a_bits,
                    (void*)&CB, (void*)&N, (void*)&B, (void*)&D, (void*)&SA, (void*)&a_kind, (void*)&a_tau,
                    (void*)&a_param, (void*)&hcp};
    cudaEvent_t e0 = g_profile.load(std::memory_order_relaxed) ? prof_start(s) : nullptr;
    GF_CUDA(cudaLaunchCooperativeKernel((const void*)k_ingest_coop, dim3((unsigned)grid), dim3(CO_T), args, 0, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e0) prof_stop("k_ingest_coop", s, e0);
    GF_CUDA(cudaStreamSynchronize(s));  // the kernel's last CTA wrote the counters to hcp
    hc = *hcp;
    static const bool timing = getenv("GF_INGEST_TIMING") != nullptr;
    if (timing && !hc.abort) {  // per-phase device time of the cooperative launch (CTA 0's view)
      static double acc[10] = {0};
      static int calls = 0;
      // A C D E F I, then E's warp part, F's chronology, plan scan and trigger scan
      const long long* t = hc.phase_ns;
      const double d[10] = {double(t[1] - t[0]), double(t[2] - t[1]), double(t[3] - t[2]), double(t[4] - t[3]),
                            double(t[5] - t[4]), double(t[6] - t[5]), double(t[7] - t[3]), double(t[8] - t[4]),
                            double(t[9] - t[8]), double(t[10] - t[9])};
      for (int i = 0; i < 10; i++) acc[i] += d[i] * 1e-3;
      if (++calls % 100 == 0) {
        fprintf(stderr, "ingest coop: %d calls, us/call A C D E F I | E.warp F.chrono F.plan F.trig:", calls);
        for (int i = 0; i < 10; i++) fprintf(stderr, " %.1f", acc[i] / calls);
        fprintf(stderr, "\n");
      }
    }
    if (!hc.abort) break;
    if (hc.abort & ABORT_NODES) {
      if (hc.minv < 0) return fail(GF_EINVAL, "node ids must be non-negative");  // storage.py:408-409
      if (hc.maxv + 1 > ((int64_t)1 << 31)) return fail(GF_EINVAL, "node ids must be < 2^31");
    }
    if ((hc.abort & ABORT_SLOW) || attempt >= 3) return GF_OK;  // the general sequence takes the batch
    if (hc.abort & ABORT_NODES) GF_TRY(grow_node_cap(g, hc.maxv + 1, s));
    if (hc.abort & ABORT_CAP) {
      GF_TRY(ensure_slots(g, g->slots_used + hc.new_slots, s));
      GF_TRY(ensure_dir(g, g->dir_used + hc.dir_need, s));
      GF_TRY(ensure_blocks(g, g->blk_used + std::max<int64_t>(0, hc.new_blocks - nfree), s));
    }
  }
  apply_ingest(g, hc, nfree, eids_user != nullptr, n, h_rej);
  *done = true;
  return GF_OK;
}

gf_status add_edges_fast(gf_graph* g, const int64_t* src_in, const int64_t* dst_in, const int64_t* ts_in, int64_t n,
                         const int64_t* eids_user, int64_t* out_user, int64_t* h_rej, cudaStream_t s) {
  if (h_rej) *h_rej = 0;
  if (n == 0) return GF_OK;
  if (n < 0 || n >= ((int64_t)1 << 30)) return fail(GF_EINVAL, "batch size must be in [0, 2^30)");
  bool done = false;
  GF_TRY(add_edges_coop(g, src_in, dst_in, ts_in, n, eids_user, out_user, h_rej, s, &done));
  if (done) return GF_OK;
  const int dir = g->directed;
  const int64_t E = dir ? n : 2 * n;
  GF_TRY(ensure_blocks(g, g->blk_used + E, s));  // new blocks <= accepted events
  if (g->node_cap == 0) GF_TRY(grow_node_cap(g, 1024, s));
  if (!g->ing_host) GF_CUDA(cudaMallocHost(&g->ing_host, 4096));
  IngestScalars* hs = (IngestScalars*)g->ing_host;
  IngestCounters* hci = (IngestCounters*)((char*)g->ing_host + 1024);  // initial counter values
  IngestCounters* hcp = (IngestCounters*)((char*)g->ing_host + 2048);  // counters read back
  memset(hci, 0, sizeof(IngestCounters));
  hci->minv = hci->tsmin = LLONG_MAX;
  hci->maxv = hci->tsmax = hci->max_eid = LLONG_MIN;
  static const bool no_graph = getenv("GF_INGEST_NO_GRAPH") != nullptr;
  const int T = 256;
  const int64_t G = 8 * num_sms();
  // handles freed by offload: their device copy is read by the commit (outside the captured graph)
  GF_TRY(stage_free_handles(g, s));
  const int64_t nfree = (int64_t)g->free_handles.size();
  IngestCounters hc;
  const auto t_start = std::chrono::steady_clock::now();
  for (int attempt = 0;; attempt++) {
    const int64_t node_cap = g->node_cap;
    const int endbit = bits_for(node_cap);
    size_t cub_bytes = 0;
    const int64_t ST = scan_tile(E);
    const int64_t tiles4 = (E + 1 + ST - 1) / ST, tiles2 = (E + ST - 1) / ST;
    {
      size_t b = 0;
      GF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                              (uint32_t*)nullptr, (int)E, 0, endbit, s));
      cub_bytes = std::max(cub_bytes, b);
      GF_CUDA(cub::DeviceScan::InclusiveSum(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, (int)E, s));
      cub_bytes = std::max(cub_bytes, b);
      GF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, (uint8_t*)nullptr, (int64_t*)nullptr, (int)n, s));
      cub_bytes = std::max(cub_bytes, b);
      GF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)(E + 1), s));
      cub_bytes = std::max(cub_bytes, b);

    }
    // scratch layout (one persistent buffer per graph)
    auto layout = [&](Arena& a, void** p) {
      size_t i = 0;
      p[i++] = a.take<IngestCounters>(1);
      p[i++] = a.take<IngestScalars>(1);
      p[i++] = a.take<longlong4>(n);  // staged edge records {src, dst, ts, eid}
      p[i++] = a.take<uint32_t>(E); p[i++] = a.take<uint32_t>(E); p[i++] = a.take<uint32_t>(E); p[i++] = a.take<uint32_t>(E);
      p[i++] = a.take<int32_t>(E); p[i++] = a.take<int32_t>(E); p[i++] = a.take<int64_t>(E + 1);
      p[i++] = a.take<uint8_t>(n); p[i++] = a.take<int64_t>(n + 1); p[i++] = a.take<int64_t>(node_cap);
      p[i++] = a.take<int64_t>(E + 1); p[i++] = a.take<int64_t>(E + 1);
      p[i++] = a.take<uint32_t>(E); p[i++] = a.take<int64_t>(E); p[i++] = a.take<int32_t>(E);
      for (int q = 0; q < 5; q++) p[i++] = a.take<int64_t>(E + 1);  // acc_cnt, cstart, fill, tail_size, nb_new
      p[i++] = a.take<longlong4>(E + 1); p[i++] = a.take<longlong4>(E + 1);  // plan4, off4
      p[i++] = a.take<int64_t>(E + 1);  // old_tail
      for (int q = 0; q < 3; q++) p[i++] = a.take<int64_t>(E + 1);  // R.first/count/cap
      p[i++] = a.take<int32_t>(E); p[i++] = a.take<uint32_t>(E);  // R.seg/key
      p[i++] = a.take<longlong2>(E); p[i++] = a.take<longlong2>(E);      // trig, tscan
      p[i++] = a.take<char>((int64_t)cub_bytes);
      p[i++] = a.take<int64_t>(tiles4 * 4); p[i++] = a.take<int64_t>(tiles4 * 4);  // plan scan agg/inc
      p[i++] = a.take<int64_t>(tiles2 * 2); p[i++] = a.take<int64_t>(tiles2 * 2);  // trigger scan agg/inc
      p[i++] = a.take<int>(2 + tiles4 + tiles2);                                  // tickets + flags (zeroed)
      return i;
    };
    void* P_[64];
    Arena probe;
    layout(probe, P_);
    const size_t need = probe.off + 4096;
    if (need > g->ing_bytes) {
      if (g->ing_buf) GF_CUDA(cudaFreeAsync(g->ing_buf, s));
      g->ing_buf = nullptr;
      g->ing_bytes = 0;
      GF_CUDA(cudaMallocAsync(&g->ing_buf, need + need / 4, s));
      g->ing_bytes = need + need / 4;
    }
    Arena A;
    A.base = (char*)g->ing_buf;
    layout(A, P_);
    int i = 0;
    IngestCounters* dc = (IngestCounters*)P_[i++];
    IngestScalars* ds = (IngestScalars*)P_[i++];
    int64_t* rec = (int64_t*)P_[i++];
    uint32_t* keys_in = (uint32_t*)P_[i++];
    uint32_t* keys = (uint32_t*)P_[i++];
    uint32_t* vals_in = (uint32_t*)P_[i++];
    uint32_t* vals = (uint32_t*)P_[i++];
    int32_t* heads = (int32_t*)P_[i++];
    int32_t* incl = (int32_t*)P_[i++];
    int64_t* seg_start = (int64_t*)P_[i++];
    uint8_t* acc = (uint8_t*)P_[i++];
    int64_t* rank = (int64_t*)P_[i++];
    int64_t* tm = (int64_t*)P_[i++];
    int64_t* keep = (int64_t*)P_[i++];
    int64_t* cpos = (int64_t*)P_[i++];
    uint32_t* ce_ev = (uint32_t*)P_[i++];
    int64_t* ce_pend = (int64_t*)P_[i++];
    int32_t* ce_seg = (int32_t*)P_[i++];
    SegPlan P;
    P.acc_cnt = (int64_t*)P_[i++];
    P.cstart = (int64_t*)P_[i++];
    P.fill = (int64_t*)P_[i++];
    P.tail_size = (int64_t*)P_[i++];
    P.nb_new = (int64_t*)P_[i++];
    P.plan4 = (longlong4*)P_[i++];
    longlong4* off4 = (longlong4*)P_[i++];
    int64_t* old_tail = (int64_t*)P_[i++];
    Recs R;
    R.first = (int64_t*)P_[i++];
    R.count = (int64_t*)P_[i++];
    R.cap = (int64_t*)P_[i++];
    R.seg = (int32_t*)P_[i++];
    R.key = (uint32_t*)P_[i++];
    longlong2* trig = (longlong2*)P_[i++];
    longlong2* tscan = (longlong2*)P_[i++];
    void* cubtmp = P_[i++];
    ScanState S4{(int64_t*)P_[i], (int64_t*)P_[i + 1], nullptr, nullptr, tiles4};
    ScanState S2{(int64_t*)P_[i + 2], (int64_t*)P_[i + 3], nullptr, nullptr, tiles2};
    int* zero = (int*)P_[i + 4];
    i += 5;
    S4.ticket = (unsigned*)zero;
    S2.ticket = (unsigned*)zero + 1;
    S4.flag = zero + 2;
    S2.flag = zero + 2 + tiles4;
    const int64_t nzero = 2 + tiles4 + tiles2;

    // per-call values: read on the device through ds
    *hs = IngestScalars{src_in, dst_in, ts_in, eids_user, out_user, g->num_nodes, g->blk_used, g->slots_used,
                        g->dir_used, g->next_edge_id, g->slot_cap - g->slots_used, g->dir_cap_total - g->dir_used,
                        g->free_dev, nfree, g->blk_cap - g->blk_used};

    // the launch sequence: identical for every call with the same key
    auto enqueue = [&](cudaStream_t s) -> gf_status {
      size_t tb = cub_bytes;
      GF_CUDA(cudaMemcpyAsync(ds, hs, sizeof(IngestScalars), cudaMemcpyHostToDevice, s));
      GF_CUDA(cudaMemcpyAsync(dc, hci, sizeof(IngestCounters), cudaMemcpyHostToDevice, s));
      GF_LAUNCH_PDL(k_stage_minmax, grid_for(std::max(n, nzero), T, G), T, 0, s, ds, n, rec, dc, zero, nzero);
      GF_LAUNCH_PDL(k_grow_nodes, grid_for(2 * n, T, G), T, 0, s, dc, ds, node_cap, g->head, g->tail, g->num_blocks,
                g->degree, g->node_valid, g->nslots, g->dir_off, g->dir_cap, g->nflags, g->nrec);
      GF_LAUNCH_PDL(k_make_events, grid_for(E, T, G), T, 0, s, rec, n, dir, keys_in, vals_in, dc, trig);
      GF_CUDA(cub::DeviceRadixSort::SortPairs(cubtmp, tb, keys_in, keys, vals_in, vals, (int)E, 0, endbit, s));
      GF_LAUNCH_PDL(k_heads, grid_for(E, T, G), T, 0, s, keys, E, heads);
      tb = cub_bytes;
      GF_CUDA(cub::DeviceScan::InclusiveSum(cubtmp, tb, heads, incl, (int)E, s));
      GF_LAUNCH_PDL(k_segments, grid_for(E, T, G), T, 0, s, keys, vals, incl, E, dir, rec, g->tail, g->bsize, g->btmax,
                seg_start, dc);
      GF_LAUNCH_PDL(k_accept, grid_for(n, T, G), T, 0, s, acc, n, tm, g->tail, g->bsize, g->btmax, dc, ds, rec, dir);
      tb = cub_bytes;
      GF_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, tb, acc, rank, (int)n, s));
      GF_LAUNCH_PDL(k_eids_keep, grid_for(std::max(n, E), T, G), T, 0, s, acc, rank, n, eids_user != nullptr, rec, dc, ds, vals, E,
                dir, keep);
      tb = cub_bytes;
      GF_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, tb, keep, cpos, (int)(E + 1), s));
      GF_LAUNCH_PDL(k_compact, grid_for(E, T, G), T, 0, s, vals, incl, cpos, keep, seg_start, E, dc, ce_ev, ce_pend, ce_seg);
      GF_LAUNCH_PDL(k_plan, grid_for(E + 1, T, G), T, 0, s, keys, seg_start, cpos, ce_pend, E, dc, g->tail, g->bsize,
                g->bcap, g->degree, g->num_blocks, g->dir_cap, g->sizing_kind, g->tau, g->sizing_param, P, old_tail);
      if (E >= SCAN_LARGE_EVENTS)
        GF_LAUNCH_PDL((k_scan_sum<4, SCAN_ITEMS_LARGE>), tiles4, SCAN_T, 0, s, (const int64_t*)P.plan4, (int64_t*)off4, E + 1, S4, dc, true);
      else
        GF_LAUNCH_PDL((k_scan_sum<4, SCAN_ITEMS_SMALL>), tiles4, SCAN_T, 0, s, (const int64_t*)P.plan4, (int64_t*)off4, E + 1, S4, dc, true);
      GF_LAUNCH_PDL(k_check_enumerate, grid_for(E, T, G), T, 0, s, off4, E, ds, dc, ce_pend, ce_ev, P, keys, seg_start,
                g->degree, g->sizing_kind, g->tau, g->sizing_param, R, trig);
      if (E >= SCAN_LARGE_EVENTS)
        GF_LAUNCH_PDL((k_scan_sum<2, SCAN_ITEMS_LARGE>), tiles2, SCAN_T, 0, s, (const int64_t*)trig, (int64_t*)tscan, E, S2, dc, false);
      else
        GF_LAUNCH_PDL((k_scan_sum<2, SCAN_ITEMS_SMALL>), tiles2, SCAN_T, 0, s, (const int64_t*)trig, (int64_t*)tscan, E, S2, dc, false);
      NodeArrays N{g->head, g->tail, g->num_blocks, g->degree, g->nslots, g->dir_off, g->dir_cap, g->node_valid,
                   g->nflags, g->nrec};
      BlockArrays B{g->bcap, g->bsize, g->btmin, g->btmax, g->bprev, g->bnext, g->bbase};
      DirArrays D{g->dir};
      GF_LAUNCH_PDL(k_commit, grid_for(E, T, G), T, 0, s, dc, ds, keys, seg_start, P, off4, R, tscan, ce_ev, rec, dir,
                old_tail, N, B, D, g->sizing_kind);
      GF_LAUNCH_PDL(k_commit_slots, grid_for(E, T, 16 * num_sms()), T, 0, s, dc, ds, keys, seg_start, P, off4, R, tscan,
                ce_ev, ce_seg, rec, dir, old_tail, g->bbase, SlotArrays{g->slots, g->sts, g->fts, g->sts32, g->fts32, g->okbits, g->node_valid});
      GF_CUDA(cudaMemcpyAsync(hcp, dc, sizeof(IngestCounters), cudaMemcpyDeviceToHost, s));
      return GF_OK;
    };

    const bool profiling = g_profile.load(std::memory_order_relaxed) != 0;
    if (no_graph || profiling) {
      GF_TRY(enqueue(s));
    } else {
      const int64_t key[8] = {E, n, (int64_t)dir | (eids_user ? 2 : 0), node_cap, g->gen, (int64_t)(intptr_t)g->ing_buf,
                              (int64_t)cub_bytes, 0};
      if (!g->ing_exec || memcmp(key, g->ing_key, sizeof(key)) != 0) {
        if (g->ing_exec) cudaGraphExecDestroy(g->ing_exec);
        g->ing_exec = nullptr;
        const uint64_t l0 = g_launches.load();
        // captured on a private stream (the caller's may be the legacy default stream)
        if (!g->cap_stream) GF_CUDA(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
        cudaGraph_t graph = nullptr;
        GF_CUDA(cudaStreamBeginCapture(g->cap_stream, cudaStreamCaptureModeThreadLocal));
        gf_status st = enqueue(g->cap_stream);
        cudaError_t ce = cudaStreamEndCapture(g->cap_stream, &graph);
        GF_TRY(st);
        if (ce != cudaSuccess) return fail(GF_ECUDA, std::string("ingest capture: ") + cudaGetErrorString(ce));
        ce = cudaGraphInstantiate(&g->ing_exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return fail(GF_ECUDA, std::string("ingest graph: ") + cudaGetErrorString(ce));
        g->ing_nodes = (int64_t)(g_launches.load() - l0);
        g_launches.fetch_sub((uint64_t)g->ing_nodes);
        memcpy(g->ing_key, key, sizeof(key));
      }
      GF_CUDA(cudaGraphLaunch(g->ing_exec, s));
      g_launches.fetch_add((uint64_t)g->ing_nodes);
    }
    const auto t_enq = std::chrono::steady_clock::now();
    GF_CUDA(cudaStreamSynchronize(s));
    hc = *hcp;
    static const bool timing = getenv("GF_INGEST_TIMING") != nullptr;
    if (timing) {
      static double enq = 0, tot = 0;
      static int calls = 0;
      const auto t_end = std::chrono::steady_clock::now();
      enq += std::chrono::duration<double, std::micro>(t_enq - t_start).count();
      tot += std::chrono::duration<double, std::micro>(t_end - t_start).count();
      if (++calls % 100 == 0)
        fprintf(stderr, "ingest: %d calls, host enqueue %.1f us/call, total %.1f us/call\n", calls, enq / calls, tot / calls);
    }
    if (!hc.abort) break;
    if (hc.minv < 0) return fail(GF_EINVAL, "node ids must be non-negative");  // storage.py:408-409
    if (hc.maxv + 1 > ((int64_t)1 << 31)) return fail(GF_EINVAL, "node ids must be < 2^31");
    if (attempt >= 3) return fail(GF_ECUDA, "ingest did not converge");
    // nothing was mutated: grow what overflowed and replay the batch
    if (hc.abort & ABORT_NODES) GF_TRY(grow_node_cap(g, hc.maxv + 1, s));
    if (hc.abort & ABORT_CAP) {
      GF_TRY(ensure_slots(g, g->slots_used + hc.new_slots, s));
      GF_TRY(ensure_dir(g, g->dir_used + hc.dir_need, s));
    }
  }
  apply_ingest(g, hc, nfree, eids_user != nullptr, n, h_rej);
  return GF_OK;
}

// ---- deletes (storage.py:479-512) ------------------------------------------
// candidate bitmap word i: slots 32i .. 32i+31 (valid edge and valid neighbour, sampling.py:178)
__global__ void k_okbits_build(const Slot* __restrict__ slots, int64_t nslots, const uint8_t* __restrict__ node_valid,
                               int64_t num_nodes, uint32_t* okbits) {
  const int64_t nw = (nslots + 31) / 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw * 32; i += (int64_t)gridDim.x * blockDim.x) {
    bool ok = false;
    if (i < nslots) {
      const Slot sl = slots[i];
      ok = sl.valid && sl.nbr >= 0 && sl.nbr < num_nodes && node_valid[sl.nbr];
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if ((threadIdx.x & 31) == 0) okbits[i >> 5] = m;
  }
}

// after a deletion: (re)build the candidate bitmap over the whole pool; its first allocation changes
// the ingest kernels' arguments, so the captured ingest graph is invalidated
gf_status okbits_rebuild(gf_graph* g, cudaStream_t s) {
  if (!g->okbits) {
    const size_t words = (size_t)(g->slot_cap + 31) / 32 + 4;  // padded: 64-bit runs read 3 words
    GF_CUDA(cudaMallocAsync(&g->okbits, sizeof(uint32_t) * words, s));
    GF_CUDA(cudaMemsetAsync(g->okbits, 0, sizeof(uint32_t) * words, s));
    g->gen++;
  }
  if (g->slots_used > 0)
    GF_LAUNCH(k_okbits_build, grid_for(g->slots_used, 256, 16 * num_sms()), 256, 0, s, g->slots, g->slots_used,
              g->node_valid, g->num_nodes, g->okbits);
  return GF_OK;
}

__global__ void k_delete_scan(Slot* slots, int64_t nslots, const int64_t* __restrict__ wanted, int64_t nw, int64_t* degree,
                              uint8_t* hit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslots; i += (int64_t)gridDim.x * blockDim.x) {
    Slot sl = slots[i];
    if (!sl.valid) continue;
    int64_t lo = 0, hi = nw;
    while (lo < hi) {
      int64_t m = (lo + hi) >> 1;
      if (wanted[m] < sl.eid) lo = m + 1;
      else hi = m;
    }
    if (lo < nw && wanted[lo] == sl.eid) {
      slots[i].valid = 0;
      atomicAdd((unsigned long long*)&degree[sl.owner], (unsigned long long)(-1LL));
      hit[lo] = 1;
    }
  }
}

__global__ void k_count_hits(const uint8_t* hit, int64_t n, long long* out) {
  long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) c += hit[i];
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)out, (unsigned long long)c);
}

__global__ void k_gather_slots(const Slot* slots, const int64_t* __restrict__ bbase, const int64_t* __restrict__ offs,
                               int64_t h0, int64_t nblk, int64_t* nbr, int64_t* eid, int64_t* ts, uint8_t* valid) {
  for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    int64_t o = offs[b], cnt = offs[b + 1] - o, base = bbase[h0 + b];
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      Slot sl = slots[base + i];
      nbr[o + i] = sl.nbr;
      eid[o + i] = sl.eid;
      ts[o + i] = sl.ts;
      valid[o + i] = (uint8_t)(sl.valid != 0);
    }
  }
}

void free_graph(gf_graph* g) {
  void* ps[] = {g->head, g->tail, g->num_blocks, g->degree, g->node_valid, g->nslots, g->dir_off, g->dir_cap,
                g->bcap, g->bsize, g->btmin, g->btmax, g->bprev, g->bnext, g->bbase, g->dir,
                g->slots, g->sts, g->fts, g->sts32, g->fts32, g->nflags, g->nrec, g->ing_buf, g->okbits,
                g->co_buf, g->co_ncnt, g->co_nseg};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (g->ing_exec) cudaGraphExecDestroy(g->ing_exec);
  if (g->ing_host) cudaFreeHost(g->ing_host);
  if (g->cap_stream) cudaStreamDestroy(g->cap_stream);
  if (g->smp_buf) cudaFree(g->smp_buf);
  if (g->free_dev) cudaFree(g->free_dev);
  if (g->smp_host) cudaFreeHost(g->smp_host);

}

}  // namespace

extern "C" {

gf_status gf_graph_create(int directed, int64_t tau, int sizing_kind, int64_t sizing_param, int device, gf_graph** out) {
  if (!out) return fail(GF_EINVAL, "out is NULL");
  *out = nullptr;
  if (sizing_kind == GF_SIZING_ADAPTIVE && tau < 1) return fail(GF_EINVAL, "tau must be >= 1");  // storage.py:85-86, 314-315
  if (sizing_kind == GF_SIZING_FIXED && sizing_param < 1) return fail(GF_EINVAL, "block size must be >= 1");
  if (sizing_kind < 0 || sizing_kind > 2) return fail(GF_EINVAL, "unknown sizing kind");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(GF_ECUDA, "no CUDA device available");
  if (device < 0 || device >= ndev) return fail(GF_EINVAL, "bad device ordinal");
  gf_graph* g = new gf_graph();
  g->device = device;
  g->directed = directed ? 1 : 0;
  g->tau = tau;
  g->sizing_kind = sizing_kind;
  g->sizing_param = sizing_param;
  *out = g;
  return GF_OK;
}

gf_status gf_graph_destroy(gf_graph* g) {
  if (!g) return GF_OK;
  DeviceGuard dg(g->device);
  cudaDeviceSynchronize();
  free_graph(g);
  delete g;
  return GF_OK;
}

gf_status gf_graph_reserve(gf_graph* g, int64_t nodes, int64_t blocks, int64_t slots, void* stream) {
  if (!g) return fail(GF_EINVAL, "graph is NULL");
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (nodes > g->node_cap) {
    g->gen++;
    int64_t k = g->num_nodes, nc = nodes;
    GF_TRY(grow_array(g->head, k, nc, s));
    GF_TRY(grow_array(g->tail, k, nc, s));
    GF_TRY(grow_array(g->num_blocks, k, nc, s));
    GF_TRY(grow_array(g->degree, k, nc, s));
    GF_TRY(grow_array(g->node_valid, k, nc, s));
    GF_TRY(grow_array(g->nslots, k, nc, s));
    GF_TRY(grow_array(g->dir_off, k, nc, s));
    GF_TRY(grow_array(g->dir_cap, k, nc, s));
    GF_TRY(grow_array(g->nflags, k, nc, s));
    GF_TRY(grow_array(g->nrec, k * NREC, nc * NREC, s));
    g->node_cap = nc;
  }
  GF_TRY(ensure_blocks(g, blocks, s));
  GF_TRY(ensure_slots(g, slots, s));
  GF_TRY(ensure_dir(g, blocks * 2, s));
  // the cooperative ingest's one-time setup (occupancy query, pinned staging, per-node counters,
  // scratch for batches of up to 2^17 edges), so that a stream's first batches do not pay it
  if (!g->ing_host) GF_CUDA(cudaMallocHost(&g->ing_host, 4096));
  const int occ = coop_occupancy();
  if (occ > 0 && g->node_cap > 0) GF_TRY(ensure_coop(g, std::min<int64_t>(std::max<int64_t>(slots, 1), 1 << 17),
                                                     (int64_t)num_sms() * occ, s));
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_graph_add_edges(gf_graph* g, const int64_t* d_src, const int64_t* d_dst, const int64_t* d_ts, int64_t n,
                             const int64_t* d_eids_in, int64_t* d_out_eids, int64_t* h_out_rejected, void* stream) {
  if (!g) return fail(GF_EINVAL, "graph is NULL");
  if (n > 0 && (!d_src || !d_dst || !d_ts || !d_out_eids)) return fail(GF_EINVAL, "NULL input array");
  DeviceGuard dg(g->device);
  return add_edges_fast(g, d_src, d_dst, d_ts, n, d_eids_in, d_out_eids, h_out_rejected, (cudaStream_t)stream);
}

gf_status gf_graph_delete_edges(gf_graph* g, const int64_t* d_eids, int64_t n, int64_t* h_out_deleted, void* stream) {
  if (!g) return fail(GF_EINVAL, "graph is NULL");
  if (h_out_deleted) *h_out_deleted = 0;
  if (n <= 0 || g->slots_used == 0) return GF_OK;
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sb(s);
  Arena A;
  {
    Arena probe;
    probe.take<int64_t>(n); probe.take<uint8_t>(n); probe.take<long long>(1);
    GF_TRY(sb.alloc(probe.off + 1024));
  }
  A.base = sb.as<char>();
  int64_t* sorted = A.take<int64_t>(n);
  uint8_t* hit = A.take<uint8_t>(n);
  long long* cnt = A.take<long long>(1);
  GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceRadixSort::SortKeys(t, b, d_eids, sorted, (int)n, 0, 64, s); }, s));
  GF_CUDA(cudaMemsetAsync(hit, 0, n, s));
  GF_CUDA(cudaMemsetAsync(cnt, 0, sizeof(long long), s));
  GF_LAUNCH(k_delete_scan, grid_for(g->slots_used, 256, 16 * num_sms()), 256, 0, s, g->slots, g->slots_used, sorted, n,
            g->degree, hit);
  GF_LAUNCH(k_count_hits, grid_for(n, 256, 4 * num_sms()), 256, 0, s, hit, n, cnt);
  long long h = 0;
  GF_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  if (h > 0) {
    g->any_deleted = 1;
    GF_TRY(okbits_rebuild(g, s));
    GF_CUDA(cudaStreamSynchronize(s));
  }
  if (h_out_deleted) *h_out_deleted = h;
  return GF_OK;
}

gf_status gf_graph_delete_node(gf_graph* g, int64_t node, int* h_out_deleted, void* stream) {
  if (!g) return fail(GF_EINVAL, "graph is NULL");
  if (h_out_deleted) *h_out_deleted = 0;
  if (node < 0 || node >= g->num_nodes) return GF_OK;
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t v = 0;
  GF_CUDA(cudaMemcpyAsync(&v, g->node_valid + node, 1, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  if (!v) return GF_OK;
  GF_CUDA(cudaMemsetAsync(g->node_valid + node, 0, 1, s));
  GF_LAUNCH(k_noderec_invalidate, 1, 1, 0, s, g->nrec, node);
  g->any_deleted = 1;
  GF_TRY(okbits_rebuild(g, s));  // every edge into the node stops being a candidate
  GF_CUDA(cudaStreamSynchronize(s));
  if (h_out_deleted) *h_out_deleted = 1;
  return GF_OK;
}

gf_status gf_graph_get_info(gf_graph* g, gf_graph_info* out) {
  if (!g || !out) return fail(GF_EINVAL, "NULL argument");
  out->num_nodes = g->num_nodes;
  out->num_block_handles = g->blk_used;
  out->live_blocks = g->blk_used - (int64_t)g->free_handles.size();
  out->slots_allocated = g->slots_used;
  out->next_edge_id = g->next_edge_id;
  out->total_edges_inserted = g->total_edges_inserted;
  out->any_deleted = g->any_deleted;
  out->directed = g->directed;
  out->tau = g->tau;
  out->sizing_kind = g->sizing_kind;
  out->sizing_param = g->sizing_param;
  out->device_bytes = g->node_cap * (8 * 7 + 2 + 8 * NREC) + g->blk_cap * 8 * 7 + g->dir_cap_total * 8 * DIRW +
                      g->slot_cap * (int64_t)(sizeof(Slot) + 8) + (g->slot_cap / FENCE + 1) * 8 + (g->slot_cap + 2 * FENCE32) * 4 + (g->slot_cap / FENCE32 + 16) * 4;
  return GF_OK;
}

gf_status gf_graph_export_nodes(gf_graph* g, int64_t* h_head, int64_t* h_tail, int64_t* h_num_blocks, int64_t* h_degree,
                                uint8_t* h_node_valid, void* stream) {
  if (!g) return fail(GF_EINVAL, "graph is NULL");
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  size_t n = (size_t)g->num_nodes;
  if (n) {
    if (h_head) GF_CUDA(cudaMemcpyAsync(h_head, g->head, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_tail) GF_CUDA(cudaMemcpyAsync(h_tail, g->tail, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_num_blocks) GF_CUDA(cudaMemcpyAsync(h_num_blocks, g->num_blocks, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_degree) GF_CUDA(cudaMemcpyAsync(h_degree, g->degree, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_node_valid) GF_CUDA(cudaMemcpyAsync(h_node_valid, g->node_valid, n, cudaMemcpyDeviceToHost, s));
  }
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_graph_export_blocks(gf_graph* g, int64_t* h_capacity, int64_t* h_size, int64_t* h_tmin, int64_t* h_tmax,
                                 int64_t* h_prev, int64_t* h_next, void* stream) {
  if (!g) return fail(GF_EINVAL, "graph is NULL");
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  size_t n = (size_t)g->blk_used;
  if (n) {
    if (h_capacity) GF_CUDA(cudaMemcpyAsync(h_capacity, g->bcap, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_size) GF_CUDA(cudaMemcpyAsync(h_size, g->bsize, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_tmin) GF_CUDA(cudaMemcpyAsync(h_tmin, g->btmin, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_tmax) GF_CUDA(cudaMemcpyAsync(h_tmax, g->btmax, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_prev) GF_CUDA(cudaMemcpyAsync(h_prev, g->bprev, 8 * n, cudaMemcpyDeviceToHost, s));
    if (h_next) GF_CUDA(cudaMemcpyAsync(h_next, g->bnext, 8 * n, cudaMemcpyDeviceToHost, s));
  }
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_graph_export_slots(gf_graph* g, int64_t h0, int64_t h1, int64_t* h_offsets, int64_t* h_nbr, int64_t* h_eid,
                                int64_t* h_ts, uint8_t* h_valid, void* stream) {
  if (!g || !h_offsets) return fail(GF_EINVAL, "NULL argument");
  if (h0 < 0 || h1 < h0 || h1 > g->blk_used) return fail(GF_EINVAL, "bad handle range");
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nb = h1 - h0;
  std::vector<int64_t> sz(nb);
  if (nb) GF_CUDA(cudaMemcpyAsync(sz.data(), g->bsize + h0, 8 * nb, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  h_offsets[0] = 0;
  for (int64_t i = 0; i < nb; i++) h_offsets[i + 1] = h_offsets[i] + sz[i];
  int64_t tot = h_offsets[nb];
  if (tot == 0) return GF_OK;
  Scratch sb(s);
  Arena A;
  GF_TRY(sb.alloc((size_t)(nb + 1) * 8 + (size_t)tot * 25 + 4096));
  A.base = sb.as<char>();
  int64_t* d_off = A.take<int64_t>(nb + 1);
  int64_t* d_nbr = A.take<int64_t>(tot);
  int64_t* d_eid = A.take<int64_t>(tot);
  int64_t* d_ts = A.take<int64_t>(tot);
  uint8_t* d_valid = A.take<uint8_t>(tot);
  GF_CUDA(cudaMemcpyAsync(d_off, h_offsets, 8 * (nb + 1), cudaMemcpyHostToDevice, s));
  GF_LAUNCH(k_gather_slots, (int)std::min<int64_t>(nb, 65535), 256, 0, s, g->slots, g->bbase, d_off, h0, nb, d_nbr, d_eid,
            d_ts, d_valid);
  if (h_nbr) GF_CUDA(cudaMemcpyAsync(h_nbr, d_nbr, 8 * tot, cudaMemcpyDeviceToHost, s));
  if (h_eid) GF_CUDA(cudaMemcpyAsync(h_eid, d_eid, 8 * tot, cudaMemcpyDeviceToHost, s));
  if (h_ts) GF_CUDA(cudaMemcpyAsync(h_ts, d_ts, 8 * tot, cudaMemcpyDeviceToHost, s));
  if (h_valid) GF_CUDA(cudaMemcpyAsync(h_valid, d_valid, tot, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

}  // extern "C"
