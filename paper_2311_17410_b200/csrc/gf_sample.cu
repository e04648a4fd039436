// gf_sample.cu -- temporal k-hop sampler (K2 + K3), one fused kernel per hop.
//
// Replaces sample_layer / _sample_one / _collect_candidates / _select and the
// sample_khop hop loop (reference sampling.py:145-299).
//
// One warp per (source, window) query.  Timestamps never decrease along a
// node's block list (storage.py:426-437 rejects out-of-order edges), so the
// in-window candidates of a query are one contiguous run [lo, hi) of list
// positions.  The warp finds hi (and lo when t_start > TS_MIN) with 32-ary
// ballot searches that probe the newest entries first: over the node's block
// directory (block tmin), then over the fence index of the boundary block,
// then one 32-timestamp window of the dense ts array.  This replaces the
// reference's tail->head block walk with block skipping (sampling.py:157-172).
//   recent:     the k newest valid candidates, newest first (sampling.py:188-190) -- bit-exact.
//   uniform/tw: k distinct candidates by Floyd's algorithm on a Philox4x32-10 stream
//               keyed by (hop seed, query key); statistically checked against the reference.
// CSR output (K3) is produced in the same kernel: each CTA claims a tile of
// queries in order, counts its samples, and obtains its output offset with a
// decoupled look-back over the preceding tiles' published counts; it then
// writes its samples.  Hop totals stay on the device, so a whole sample_khop
// is a fixed sequence of launches with one host synchronisation at the end.
#include <cub/cub.cuh>
#include <cuda/atomic>

#include <algorithm>
#include <vector>

#include "gf_graph.cuh"

using namespace gf;

namespace {

constexpr int WARPS = 8;
constexpr int THREADS = WARPS * 32;
constexpr int QW = 4;              // queries per warp per tile
constexpr int TQ = WARPS * QW;     // queries per tile (== 32: one per lane of the scanning warp)
static_assert(TQ == 32, "tile scan assumes 32 queries per tile");

constexpr unsigned long long FLAG_A = 1ull << 62;  // tile aggregate published
constexpr unsigned long long FLAG_P = 2ull << 62;  // tile inclusive prefix published
constexpr unsigned long long VAL_MASK = (1ull << 62) - 1;

__device__ __forceinline__ bool node_ok(const GraphView& G, int64_t v) {
  return v >= 0 && v < G.num_nodes && G.node_valid[v];
}

// number of timestamps < x in the block whose slots are sts[base, base + size)
__device__ __forceinline__ int64_t block_lower_bound(const GraphView& G, int64_t base, int64_t size, int64_t x) {
  const int lane = lane_id();
  int64_t seg_lo, seg_hi;
  int64_t f0 = (base + FENCE - 1) / FENCE, f1 = (base + size - 1) / FENCE;  // fences inside the block
  if (size <= FENCE || f0 > f1) {
    seg_lo = base;
    seg_hi = base + size;
  } else {
    int64_t j = warp_lower_bound(G.fts + f0, 1, f1 - f0 + 1, x);  // fences < x
    if (j == 0) {
      seg_lo = base;
      seg_hi = f0 * FENCE;
    } else {
      seg_lo = (f0 + j - 1) * FENCE;
      seg_hi = min(seg_lo + FENCE, base + size);
    }
  }
  // seg length <= 2 * FENCE - 1 only when size <= FENCE... otherwise <= FENCE
  int64_t cnt = 0;
  for (int64_t p0 = seg_lo; p0 < seg_hi; p0 += 32) {
    int64_t p = p0 + lane;
    bool lt = p < seg_hi && __ldg(G.sts + p) < x;
    unsigned m = __ballot_sync(0xffffffffu, lt);
    cnt += __popc(m);
    if (m != 0xffffffffu) break;
  }
  return seg_lo - base + cnt;
}

struct Bound {
  int64_t pos;  // list position (count of slots with ts < x)
  int64_t blk;  // directory index of the block holding pos - 1 (or -1)
};

// list position of the first slot with ts >= x, and the block holding the slot before it
__device__ __forceinline__ Bound list_lower_bound(const GraphView& G, int64_t d0, int64_t nb, int64_t ns_end, int64_t x) {
  int64_t B = warp_lower_bound(G.dtmin + d0, 1, nb, x);  // blocks with tmin < x
  if (B == 0) return Bound{__ldg(G.dcum + d0), -1};
  int64_t b = B - 1;
  int64_t cum = __ldg(G.dcum + d0 + b);
  int64_t size = (b == nb - 1) ? (ns_end - cum) : (__ldg(G.dcum + d0 + b + 1) - cum);
  int64_t in = block_lower_bound(G, __ldg(G.dbase + d0 + b), size, x);
  // in >= 1 because tmin_b < x; the slot before the boundary is in block b
  return Bound{cum + in, b};
}

// directory index of the block holding list position p
__device__ __forceinline__ int64_t block_of(const GraphView& G, bool regular, int64_t d0, int64_t nb, int64_t p) {
  if (regular) {
    const SizingLaw& L = G.law;
    if (L.kind == GF_SIZING_FIXED) return p / L.size;
    if (p >= L.cum_m) return L.m + (p - L.cum_m) / L.tau;
    return p == 0 ? 0 : 64 - __clzll(p);
  }
  return upper_bound_seq(G.dcum + d0, nb, p) - 1;
}

__device__ __forceinline__ Slot load_slot(const Slot* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  int4 a = __ldg(q), b = __ldg(q + 1);
  Slot s;
  s.ts = ((int64_t)(uint32_t)a.y << 32) | (uint32_t)a.x;
  s.eid = ((int64_t)(uint32_t)a.w << 32) | (uint32_t)a.z;
  s.nbr = b.x;
  s.owner = b.y;
  s.valid = (uint32_t)b.z;
  s.pad = 0;
  return s;
}

__device__ __forceinline__ bool slot_ok(const GraphView& G, const Slot& s) {
  return s.valid && G.node_valid[s.nbr];
}

__device__ __forceinline__ int nth_set_bit(unsigned m, int n) {  // 0-based
  for (int i = 0; i < n; i++) m &= m - 1;
  return __ffs(m) - 1;
}

struct HopArgs {
  GraphView G;
  const int64_t* src;
  const int64_t* t_start;  // NULL => TS_MIN
  const int64_t* t_end;
  const uint64_t* keys;    // NULL => key_base + q
  uint64_t key_base;
  int64_t n;               // query count when n_dev == NULL
  const int64_t* n_dev;    // device query count (previous hop's total)
  int64_t fanout;
  int policy;
  int64_t delta;
  uint64_t seed;
  int64_t* offsets;        // n + 1
  int64_t* nbr;
  int64_t* eid;
  int64_t* ts;
  uint64_t* out_keys;      // optional child keys
  int64_t out_cap;
  unsigned long long* tile_state;
  unsigned int* tile_counter;
  int64_t* total;          // this hop's total (device)
  int* overflow;           // set when a write would exceed out_cap
};

__device__ __forceinline__ void emit(const HopArgs& A, int64_t at, const Slot& s, uint64_t qkey, int64_t i) {
  if (at >= A.out_cap) {
    *A.overflow = 1;
    return;
  }
  __stcs((long long*)A.nbr + at, (long long)s.nbr);
  __stcs((long long*)A.eid + at, (long long)s.eid);
  __stcs((long long*)A.ts + at, (long long)s.ts);
  if (A.out_keys) __stcs((long long*)A.out_keys + at, (long long)child_key(qkey, (uint64_t)i));
}

// ---- phase 1: window search + candidate count ---------------------------------
struct QState {
  int64_t lo, hi, nv, k;
  int64_t blk;  // block holding hi - 1
};

__device__ __forceinline__ QState search_query(const HopArgs& A, int64_t q) {
  const GraphView& G = A.G;
  const int lane = lane_id();
  QState S{0, 0, 0, 0, -1};
  int64_t v = A.src[q];
  if (!node_ok(G, v)) return S;  // sampling.py:153-155
  int64_t nb = G.num_blocks[v];
  if (nb == 0) return S;
  int64_t te = A.t_end[q];
  int64_t tsr = A.t_start ? A.t_start[q] : GF_TS_MIN;
  if (A.policy == GF_POLICY_TIME_WINDOW) tsr = (te < GF_TS_MIN + A.delta) ? GF_TS_MIN : te - A.delta;  // sampling.py:202-203
  int64_t d0 = G.dir_off[v], ns = G.nslots[v];
  Bound h = list_lower_bound(G, d0, nb, ns, te);
  int64_t lo = (tsr == GF_TS_MIN) ? __ldg(G.dcum + d0) : list_lower_bound(G, d0, nb, ns, tsr).pos;
  if (h.pos <= lo) {
    S.lo = S.hi = lo;
    return S;
  }
  S.lo = lo;
  S.hi = h.pos;
  S.blk = h.blk;
  if (!G.any_deleted) {
    S.nv = h.pos - lo;
  } else {
    // valid candidates only (valid edge && valid neighbour, sampling.py:178); recent needs <= fanout
    int64_t limit = (A.policy == GF_POLICY_RECENT) ? A.fanout : INT64_MAX;
    int64_t b = h.blk, p = h.pos, cnt = 0;
    while (p > lo && cnt < limit) {
      int64_t cum = __ldg(G.dcum + d0 + b);
      int64_t cst = max(max(cum, lo), p - 32);
      int64_t pos = p - 1 - lane;
      bool ok = false;
      if (pos >= cst) ok = slot_ok(G, load_slot(G.slots + __ldg(G.dbase + d0 + b) + (pos - cum)));
      cnt += __popc(__ballot_sync(0xffffffffu, ok));
      p = cst;
      if (p == cum) b--;
    }
    S.nv = cnt < limit ? cnt : limit;
  }
  S.k = S.nv < A.fanout ? S.nv : A.fanout;
  return S;
}

// ---- phase 2: selection + write -------------------------------------------------
__device__ __forceinline__ void emit_query(const HopArgs& A, int64_t q, const QState& S, int64_t out) {
  const GraphView& G = A.G;
  const int lane = lane_id();
  const int64_t k = S.k;
  int64_t v = A.src[q];
  int64_t d0 = G.dir_off[v], nb = G.num_blocks[v];
  uint64_t qkey = A.keys ? A.keys[q] : A.key_base + (uint64_t)q;
  const int64_t lo = S.lo, hi = S.hi, nv = S.nv;
  if (A.policy == GF_POLICY_RECENT || k == nv) {
    // newest first: the first k valid candidates walking back from hi - 1
    const unsigned lt = (1u << lane) - 1u;
    int64_t b = S.blk, p = hi, done = 0;
    while (done < k && p > lo) {
      int64_t cum = __ldg(G.dcum + d0 + b);
      int64_t cst = max(max(cum, lo), p - 32);
      int64_t pos = p - 1 - lane;
      bool ok = false;
      Slot s;
      if (pos >= cst) {
        s = load_slot(G.slots + __ldg(G.dbase + d0 + b) + (pos - cum));
        ok = G.any_deleted ? slot_ok(G, s) : true;
      }
      unsigned m = __ballot_sync(0xffffffffu, ok);
      int64_t r = done + __popc(m & lt);
      if (ok && r < k) emit(A, out + r, s, qkey, r);
      done += __popc(m);
      p = cst;
      if (p == cum) b--;
    }
    return;
  }
  const bool regular = !(G.nflags[v] & 1);
  if (k <= 32) {
    // Floyd: draw t_i in [0, nv-k+i] (independent draws, one per lane), then dedupe in order
    int64_t t = 0;
    if (lane < k) t = (int64_t)bounded64(rand64(A.seed, qkey, (uint64_t)lane), (uint64_t)(nv - k + lane + 1));
    int64_t mine = -1;
    for (int i = 0; i < (int)k; i++) {
      int64_t ti = __shfl_sync(0xffffffffu, t, i);
      bool dup = __ballot_sync(0xffffffffu, lane < i && mine == ti) != 0;
      if (lane == i) mine = dup ? (nv - k + i) : ti;
    }
    if (!G.any_deleted) {
      if (lane < k) {
        int64_t p = lo + mine;
        int64_t b = block_of(G, regular, d0, nb, p);
        emit(A, out + lane, load_slot(G.slots + __ldg(G.dbase + d0 + b) + (p - __ldg(G.dcum + d0 + b))), qkey, lane);
      }
    } else {
      // chronological valid rank -> position: forward scan over [lo, hi)
      int64_t b = block_of(G, false, d0, nb, lo);
      int64_t p = lo, rank0 = 0;
      while (p < hi) {
        int64_t cum = __ldg(G.dcum + d0 + b);
        int64_t bend = (b == nb - 1) ? G.nslots[v] : __ldg(G.dcum + d0 + b + 1);
        int64_t cen = min(min(bend, hi), p + 32);
        int64_t pos = p + lane;
        Slot s;
        s.ts = 0; s.eid = 0; s.nbr = 0;
        bool ok = false;
        if (pos < cen) {
          s = load_slot(G.slots + __ldg(G.dbase + d0 + b) + (pos - cum));
          ok = slot_ok(G, s);
        }
        unsigned m = __ballot_sync(0xffffffffu, ok);
        int c = __popc(m);
        bool here = lane < k && mine >= rank0 && mine < rank0 + c;
        int srcl = here ? nth_set_bit(m, (int)(mine - rank0)) : lane;
        Slot t2;
        t2.ts = __shfl_sync(0xffffffffu, s.ts, srcl);
        t2.eid = __shfl_sync(0xffffffffu, s.eid, srcl);
        t2.nbr = __shfl_sync(0xffffffffu, s.nbr, srcl);
        if (here) emit(A, out + lane, t2, qkey, lane);
        rank0 += c;
        p = cen;
        if (p == bend) b++;
      }
    }
    return;
  }
  // large fanout: keep the Floyd set in the output's eid column while drawing
  if (out + k > A.out_cap) {
    if (lane == 0) *A.overflow = 1;
    return;
  }
  int64_t* sel = A.eid + out;
  for (int64_t i = 0; i < k; i++) {
    int64_t j = nv - k + i;
    int64_t ti = (int64_t)bounded64(rand64(A.seed, qkey, (uint64_t)i), (uint64_t)(j + 1));
    bool dup = false;
    for (int64_t c0 = 0; c0 < i; c0 += 32) {
      int64_t c = c0 + lane;
      if (__ballot_sync(0xffffffffu, c < i && sel[c] == ti)) dup = true;
    }
    __syncwarp();
    if (lane == 0) sel[i] = dup ? j : ti;
    __syncwarp();
  }
  for (int64_t i0 = 0; i0 < k; i0 += 32) {
    int64_t i = i0 + lane;
    int64_t rk = (i < k) ? sel[i] : -1;
    __syncwarp();
    if (!G.any_deleted) {
      if (i < k) {
        int64_t p = lo + rk;
        int64_t b = block_of(G, regular, d0, nb, p);
        emit(A, out + i, load_slot(G.slots + __ldg(G.dbase + d0 + b) + (p - __ldg(G.dcum + d0 + b))), qkey, i);
      }
    } else {
      for (int l = 0; l < 32 && i0 + l < k; l++) {
        int64_t want = __shfl_sync(0xffffffffu, rk, l);
        int64_t p = lo, seen = 0;
        int64_t b = block_of(G, false, d0, nb, lo);
        while (p < hi) {
          int64_t cum = __ldg(G.dcum + d0 + b);
          int64_t bend = (b == nb - 1) ? G.nslots[v] : __ldg(G.dcum + d0 + b + 1);
          int64_t cen = min(min(bend, hi), p + 32);
          int64_t pos = p + lane;
          Slot s;
          s.ts = 0; s.eid = 0; s.nbr = 0;
          bool ok = false;
          if (pos < cen) {
            s = load_slot(G.slots + __ldg(G.dbase + d0 + b) + (pos - cum));
            ok = slot_ok(G, s);
          }
          unsigned m = __ballot_sync(0xffffffffu, ok);
          int c = __popc(m);
          if (want < seen + c) {
            int srcl = nth_set_bit(m, (int)(want - seen));
            Slot t2;
            t2.ts = __shfl_sync(0xffffffffu, s.ts, srcl);
            t2.eid = __shfl_sync(0xffffffffu, s.eid, srcl);
            t2.nbr = __shfl_sync(0xffffffffu, s.nbr, srcl);
            if (lane == 0) emit(A, out + i0 + l, t2, qkey, i0 + l);
            break;
          }
          seen += c;
          p = cen;
          if (p == bend) b++;
        }
      }
    }
    __syncwarp();
  }
}

// ---- the fused hop kernel ----------------------------------------------------------
__global__ void __launch_bounds__(THREADS, 4) k_sample_hop(HopArgs A) {
  __shared__ int64_t s_lo[TQ], s_hi[TQ], s_nv[TQ], s_k[TQ], s_blk[TQ], s_excl[TQ];
  __shared__ int64_t s_base;
  __shared__ unsigned int s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t n = A.n_dev ? *A.n_dev : A.n;
  if (*A.overflow) n = 0;  // a previous hop overflowed: its outputs are incomplete
  const int64_t ntiles = (n + TQ - 1) / TQ;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(A.tile_counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
    // phase 1
    for (int j = 0; j < QW; j++) {
      int idx = warp * QW + j;
      int64_t q = tile * TQ + idx;
      QState S{0, 0, 0, 0, -1};
      if (q < n) S = search_query(A, q);
      if (lane == 0) {
        s_lo[idx] = S.lo;
        s_hi[idx] = S.hi;
        s_nv[idx] = S.nv;
        s_k[idx] = S.k;
        s_blk[idx] = S.blk;
      }
    }
    __syncthreads();
    // tile scan + decoupled look-back (warp 0)
    if (warp == 0) {
      int64_t c = s_k[lane], incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      s_excl[lane] = incl - c;
      int64_t agg = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 0) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> mine(A.tile_state[tile]);
        int64_t excl = 0;
        if (tile == 0) {
          mine.store(FLAG_P | (unsigned long long)agg, cuda::memory_order_release);
        } else {
          mine.store(FLAG_A | (unsigned long long)agg, cuda::memory_order_release);
          int64_t t = tile - 1;
          while (true) {
            cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> pred(A.tile_state[t]);
            unsigned long long st = pred.load(cuda::memory_order_acquire);
            if ((st >> 62) == 0) continue;
            excl += (int64_t)(st & VAL_MASK);
            if ((st >> 62) == 2) break;
            t--;
          }
          mine.store(FLAG_P | (unsigned long long)(excl + agg), cuda::memory_order_release);
        }
        s_base = excl;
        if (tile == ntiles - 1) *A.total = excl + agg;
        if (tile == 0) A.offsets[0] = 0;
      }
    }
    __syncthreads();
    // phase 2
    const int64_t base = s_base;
    for (int j = 0; j < QW; j++) {
      int idx = warp * QW + j;
      int64_t q = tile * TQ + idx;
      if (q >= n) break;
      int64_t out = base + s_excl[idx];
      QState S{s_lo[idx], s_hi[idx], s_nv[idx], s_k[idx], s_blk[idx]};
      if (lane == 0) A.offsets[q + 1] = out + S.k;
      if (S.k > 0) emit_query(A, q, S, out);
    }
    __syncthreads();
  }
}

__global__ void k_zero_total(int64_t* total, int64_t* offsets) {
  // a hop with no queries has total 0 and offsets[0] = 0
  *total = 0;
  offsets[0] = 0;
}

int64_t persistent_grid() {
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sample_hop, THREADS, 0);
    if (per_sm <= 0) per_sm = 1;
  }
  return (int64_t)num_sms() * per_sm;
}

gf_status check_args(int64_t n, int64_t fanout, int policy, int64_t delta) {
  if (n < 0) return fail(GF_EINVAL, "negative query count");
  if (fanout < 1) return fail(GF_EINVAL, "fanout must be >= 1");                 // sampling.py:240-241
  if (policy < 0 || policy > 2) return fail(GF_EINVAL, "unknown policy kind");   // sampling.py:38-39
  if (policy == GF_POLICY_TIME_WINDOW && delta <= 0) return fail(GF_EINVAL, "time_window policy requires delta > 0");
  return GF_OK;
}

// Launch one hop.  `state` is tile bookkeeping for at most max_q queries.
gf_status launch_hop(HopArgs A, int64_t max_q, unsigned long long* state, cudaStream_t s) {
  int64_t max_tiles = (max_q + TQ - 1) / TQ;
  A.tile_state = state + 1;
  A.tile_counter = reinterpret_cast<unsigned int*>(state);
  GF_CUDA(cudaMemsetAsync(state, 0, sizeof(unsigned long long) * (size_t)(max_tiles + 1), s));
  GF_LAUNCH(k_zero_total, 1, 1, 0, s, A.total, A.offsets);
  int64_t grid = std::min<int64_t>(persistent_grid(), std::max<int64_t>(max_tiles, 1));
  GF_LAUNCH(k_sample_hop, grid, THREADS, 0, s, A);
  return GF_OK;
}

}  // namespace

extern "C" {

gf_status gf_sample_layer(gf_graph* g, const int64_t* d_src, const int64_t* d_t_start, const int64_t* d_t_end, int64_t n,
                          int64_t fanout, int policy, int64_t delta, uint64_t seed, const uint64_t* d_keys,
                          uint64_t key_base, int64_t* d_offsets, int64_t* d_nbr, int64_t* d_eid, int64_t* d_ts,
                          uint64_t* d_out_keys, int64_t out_cap, int64_t* h_out_total, void* stream) {
  if (!g || !h_out_total || !d_offsets) return fail(GF_EINVAL, "NULL argument");
  GF_TRY(check_args(n, fanout, policy, delta));
  if (n >= ((int64_t)1 << 40)) return fail(GF_EINVAL, "too many queries in one call");
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  *h_out_total = 0;
  if (n == 0) {
    GF_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), s));
    return GF_OK;
  }
  int64_t max_tiles = (n + TQ - 1) / TQ;
  Scratch sb(s);
  GF_TRY(sb.alloc(sizeof(unsigned long long) * (size_t)(max_tiles + 1) + 64));
  unsigned long long* state = sb.as<unsigned long long>();
  int64_t* total = reinterpret_cast<int64_t*>(state + max_tiles + 1);
  int* overflow = reinterpret_cast<int*>(total + 1);
  GF_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int), s));
  HopArgs A{view_of(g), d_src, d_t_start, d_t_end, d_keys, key_base, n, nullptr, fanout, policy, delta, seed,
            d_offsets, d_nbr, d_eid, d_ts, d_out_keys, out_cap, nullptr, nullptr, total, overflow};
  GF_TRY(launch_hop(A, n, state, s));
  int64_t h[2] = {0, 0};
  GF_CUDA(cudaMemcpyAsync(h, total, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  *h_out_total = h[0];
  if (*reinterpret_cast<int*>(&h[1]) || h[0] > out_cap) return fail(GF_ERANGE, "output buffer too small");
  return GF_OK;
}

gf_status gf_sample_khop(gf_graph* g, const int64_t* d_roots, const int64_t* d_ts, int64_t n_roots, const int64_t* h_fanouts,
                         int n_hops, int policy, int64_t delta, uint64_t seed, uint64_t root_key_base,
                         int64_t* const* d_offsets, int64_t* const* d_nbr, int64_t* const* d_eid, int64_t* const* d_ts_out,
                         const int64_t* h_caps, int64_t* h_totals, void* stream) {
  if (!g || (n_hops > 0 && (!h_fanouts || !d_offsets || !d_nbr || !d_eid || !d_ts_out || !h_caps || !h_totals)))
    return fail(GF_EINVAL, "NULL argument");
  if (n_roots < 0) return fail(GF_EINVAL, "negative root count");
  for (int h = 0; h < n_hops; h++) {
    GF_TRY(check_args(n_roots, h_fanouts[h], policy, delta));  // SampleRequest.validate, sampling.py:64-68
    if (h_caps[h] < 0) return fail(GF_EINVAL, "negative capacity");
    h_totals[h] = 0;
  }
  if (n_hops == 0) return GF_OK;
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  const bool need_keys = policy != GF_POLICY_RECENT;
  // scratch: tile state (sized for the largest hop), per-hop totals + overflow flag, key buffers
  int64_t max_q = n_roots;
  for (int h = 0; h + 1 < n_hops; h++) max_q = std::max(max_q, h_caps[h]);
  int64_t max_tiles = (max_q + TQ - 1) / TQ;
  int64_t key_cap = 0;
  if (need_keys)
    for (int h = 0; h + 1 < n_hops; h++) key_cap = std::max(key_cap, h_caps[h]);
  Scratch sb(s);
  Arena Ar;
  {
    Arena probe;
    probe.take<unsigned long long>(max_tiles + 1);
    probe.take<int64_t>(n_hops + 2);
    probe.take<uint64_t>(key_cap);
    probe.take<uint64_t>(key_cap);
    GF_TRY(sb.alloc(probe.off + 1024));
  }
  Ar.base = sb.as<char>();
  unsigned long long* state = Ar.take<unsigned long long>(max_tiles + 1);
  int64_t* totals = Ar.take<int64_t>(n_hops + 2);
  uint64_t* keybuf[2] = {Ar.take<uint64_t>(key_cap), Ar.take<uint64_t>(key_cap)};
  int* overflow = reinterpret_cast<int*>(totals + n_hops);
  GF_CUDA(cudaMemsetAsync(totals, 0, sizeof(int64_t) * (n_hops + 2), s));
  const int64_t* src = d_roots;
  const int64_t* tend = d_ts;
  const int64_t* n_dev = nullptr;
  const uint64_t* in_keys = nullptr;
  for (int h = 0; h < n_hops; h++) {
    uint64_t* out_keys = (need_keys && h + 1 < n_hops) ? keybuf[h & 1] : nullptr;
    int64_t hop_max_q = (h == 0) ? n_roots : h_caps[h - 1];
    HopArgs A{view_of(g), src, nullptr, tend, in_keys, root_key_base, n_roots, n_dev, h_fanouts[h], policy, delta,
              gf::seed_sequence_2(seed, h), d_offsets[h], d_nbr[h], d_eid[h], d_ts_out[h], out_keys, h_caps[h],
              nullptr, nullptr, totals + h, overflow};
    GF_TRY(launch_hop(A, hop_max_q, state, s));
    src = d_nbr[h];
    tend = d_ts_out[h];
    n_dev = totals + h;
    in_keys = out_keys;
  }
  std::vector<int64_t> h(n_hops + 1);
  GF_CUDA(cudaMemcpyAsync(h.data(), totals, sizeof(int64_t) * (n_hops + 1), cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < n_hops; i++) h_totals[i] = h[i];
  if (*reinterpret_cast<int*>(&h[n_hops])) return fail(GF_ERANGE, "output buffer too small");
  for (int i = 0; i < n_hops; i++)
    if (h[i] > h_caps[i]) return fail(GF_ERANGE, "output buffer too small");
  return GF_OK;
}

}  // extern "C"
