// gf_sample.cu -- temporal k-hop sampler (K2 + K3).
//
// Replaces sample_layer / _sample_one / _collect_candidates / _select and the
// sample_khop hop loop (reference sampling.py:145-299).
//
// One warp per (source, window) query.  Because timestamps never decrease
// along a node's block list (storage.py:426-437 rejects out-of-order edges),
// the in-window candidates of a query are one contiguous run [lo, hi) of
// list positions.  The warp finds hi (and lo when t_start > TS_MIN) with two
// 32-ary ballot searches: over the node's block directory (tmin per block,
// newest blocks probed first) and then inside the boundary block.  This is
// the reference's tail->head block walk with block skipping (sampling.py:157-172)
// without the pointer chase.
//   recent:       the k newest valid candidates, newest first (sampling.py:188-190) -- bit-exact.
//   uniform/tw:   k distinct candidates by Floyd's algorithm on a Philox4x32-10
//                 stream keyed by (hop seed, query key) -- statistically checked.
// Output is CSR: pass A counts per query, a device scan makes offsets, pass
// B writes neighbours/edge ids/timestamps (K3 compaction by count-then-write).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "gf_graph.cuh"

using namespace gf;

namespace {

constexpr int WARPS_PER_BLOCK = 8;
constexpr int THREADS = WARPS_PER_BLOCK * 32;

__device__ __forceinline__ bool node_ok(const GraphView& G, int64_t v) {
  return v >= 0 && v < G.num_nodes && G.node_valid[v];
}

__device__ __forceinline__ const int64_t* slot_ts_ptr(const GraphView& G, int64_t base) {
  return &G.slots[base].ts;
}

// number of list slots of the node with ts < x (absolute list position)
__device__ __forceinline__ int64_t list_lower_bound(const GraphView& G, int64_t d0, int64_t nb, int64_t ns_end, int64_t x) {
  int64_t B = warp_lower_bound(G.dtmin + d0, 1, nb, x);
  if (B == 0) return __ldg(G.dcum + d0);
  int64_t b = B - 1;
  int64_t cum = __ldg(G.dcum + d0 + b);
  int64_t size = (b == nb - 1) ? (ns_end - cum) : (__ldg(G.dcum + d0 + b + 1) - cum);
  int64_t base = __ldg(G.dbase + d0 + b);
  return cum + warp_lower_bound(slot_ts_ptr(G, base), 4, size, x);
}

// block index (0-based in the node's directory) containing list position p
__device__ __forceinline__ int64_t warp_block_of(const GraphView& G, int64_t d0, int64_t nb, int64_t p) {
  return warp_lower_bound(G.dcum + d0, 1, nb, p + 1) - 1;
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

struct QueryIn {
  const int64_t* src;
  const int64_t* t_start;  // NULL => TS_MIN
  const int64_t* t_end;
  const uint64_t* keys;    // NULL => key_base + q
  uint64_t key_base;
  int64_t n;
  int64_t fanout;
  int policy;
  int64_t delta;
  uint64_t seed;
};

struct QueryScratch {
  int64_t* lo;
  int64_t* hi;
  int64_t* nv;  // number of candidates the selection runs over
};

// ---- pass A: window search + counts --------------------------------------------
__global__ void __launch_bounds__(THREADS, 4) k_sample_count(GraphView G, QueryIn Q, QueryScratch S, int64_t* counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = warp; q < Q.n; q += nwarps) {
    int64_t v = Q.src[q];
    int64_t te = Q.t_end[q];
    int64_t tsr = Q.t_start ? Q.t_start[q] : GF_TS_MIN;
    if (Q.policy == GF_POLICY_TIME_WINDOW) tsr = (te < GF_TS_MIN + Q.delta) ? GF_TS_MIN : te - Q.delta;  // sampling.py:202-203
    int64_t lo = 0, hi = 0, nv = 0, k = 0;
    if (node_ok(G, v)) {  // sampling.py:153-155
      int64_t nb = G.num_blocks[v];
      if (nb > 0) {
        int64_t d0 = G.dir_off[v], ns = G.nslots[v];
        hi = list_lower_bound(G, d0, nb, ns, te);
        lo = (tsr == GF_TS_MIN) ? __ldg(G.dcum + d0) : list_lower_bound(G, d0, nb, ns, tsr);
        if (hi > lo) {
          if (!G.any_deleted) {
            nv = hi - lo;
          } else {
            // count valid candidates (valid edge && valid neighbour, sampling.py:178);
            // recent needs at most `fanout` of them
            int64_t limit = (Q.policy == GF_POLICY_RECENT) ? Q.fanout : INT64_MAX;
            int64_t b = warp_block_of(G, d0, nb, hi - 1);
            int64_t p = hi, cnt = 0;
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
            nv = cnt < limit ? cnt : limit;
          }
          k = nv < Q.fanout ? nv : Q.fanout;
        } else {
          hi = lo;
        }
      }
    }
    if (lane == 0) {
      S.lo[q] = lo;
      S.hi[q] = hi;
      S.nv[q] = nv;
      counts[q] = k;
    }
  }
}

struct LayerOut {
  const int64_t* offsets;
  int64_t* nbr;
  int64_t* eid;
  int64_t* ts;
  uint64_t* keys;  // optional child keys
};

__device__ __forceinline__ void emit(const LayerOut& O, int64_t at, const Slot& s, uint64_t qkey, int64_t i) {
  O.nbr[at] = s.nbr;
  O.eid[at] = s.eid;
  O.ts[at] = s.ts;
  if (O.keys) O.keys[at] = child_key(qkey, (uint64_t)i);
}

// newest-first walk emitting the first k valid candidates of [lo, hi)
__device__ __forceinline__ void emit_recent(const GraphView& G, int64_t d0, int64_t nb, int64_t lo, int64_t hi, int64_t k,
                                            const LayerOut& O, int64_t out, uint64_t qkey) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int64_t b = warp_block_of(G, d0, nb, hi - 1);
  int64_t p = hi, done = 0;
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
    if (ok && r < k) emit(O, out + r, s, qkey, r);
    done += __popc(m);
    p = cst;
    if (p == cum) b--;
  }
}

// map a list position to its slot (per-lane binary search over the directory)
__device__ __forceinline__ const Slot* slot_at(const GraphView& G, int64_t d0, int64_t nb, int64_t p) {
  int64_t b = upper_bound_seq(G.dcum + d0, nb, p) - 1;
  return G.slots + __ldg(G.dbase + d0 + b) + (p - __ldg(G.dcum + d0 + b));
}

// ---- pass B: selection + CSR write ---------------------------------------------
__global__ void __launch_bounds__(THREADS, 4) k_sample_write(GraphView G, QueryIn Q, QueryScratch S, LayerOut O) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = warp; q < Q.n; q += nwarps) {
    int64_t out = O.offsets[q];
    int64_t k = O.offsets[q + 1] - out;
    if (k == 0) continue;
    int64_t v = Q.src[q];
    int64_t lo = S.lo[q], hi = S.hi[q], nv = S.nv[q];
    int64_t d0 = G.dir_off[v], nb = G.num_blocks[v];
    uint64_t qkey = Q.keys ? Q.keys[q] : Q.key_base + (uint64_t)q;
    if (Q.policy == GF_POLICY_RECENT || k == nv) {
      emit_recent(G, d0, nb, lo, hi, k, O, out, qkey);
      continue;
    }
    // uniform / time_window with k < nv: Floyd's k-of-nv on the Philox stream
    if (k <= 32) {
      int64_t t = 0;
      if (lane < k) t = (int64_t)bounded64(rand64(Q.seed, qkey, (uint64_t)lane), (uint64_t)(nv - k + lane + 1));
      int64_t mine = -1;
      for (int i = 0; i < k; i++) {
        int64_t ti = __shfl_sync(0xffffffffu, t, i);
        bool dup = __ballot_sync(0xffffffffu, lane < i && mine == ti) != 0;
        if (lane == i) mine = dup ? (nv - k + i) : ti;
      }
      if (!G.any_deleted) {
        if (lane < k) emit(O, out + lane, load_slot(slot_at(G, d0, nb, lo + mine)), qkey, lane);
      } else {
        // chronological valid rank -> position: forward scan over [lo, hi)
        int64_t b = warp_block_of(G, d0, nb, lo);
        int64_t p = lo, rank0 = 0;
        while (p < hi) {
          int64_t cum = __ldg(G.dcum + d0 + b);
          int64_t bend = (b == nb - 1) ? G.nslots[v] : __ldg(G.dcum + d0 + b + 1);
          int64_t cen = min(min(bend, hi), p + 32);
          int64_t pos = p + lane;
          Slot s;
          bool ok = false;
          if (pos < cen) {
            s = load_slot(G.slots + __ldg(G.dbase + d0 + b) + (pos - cum));
            ok = slot_ok(G, s);
          }
          unsigned m = __ballot_sync(0xffffffffu, ok);
          int c = __popc(m);
          bool mine_here = lane < k && mine >= rank0 && mine < rank0 + c;
          int srcl = mine_here ? (__fns(m, 0, (int)(mine - rank0) + 1)) : lane;
          Slot t2;
          t2.ts = __shfl_sync(0xffffffffu, s.ts, srcl);
          t2.eid = __shfl_sync(0xffffffffu, s.eid, srcl);
          t2.nbr = __shfl_sync(0xffffffffu, s.nbr, srcl);
          if (mine_here) emit(O, out + lane, t2, qkey, lane);
          rank0 += c;
          p = cen;
          if (p == bend) b++;
        }
      }
    } else {
      // large fanout: keep the Floyd set in the output (eid column) while drawing
      int64_t* sel = O.eid + out;
      for (int64_t i = 0; i < k; i++) {
        int64_t j = nv - k + i;
        int64_t ti = (int64_t)bounded64(rand64(Q.seed, qkey, (uint64_t)i), (uint64_t)(j + 1));
        bool dup = false;
        for (int64_t c0 = 0; c0 < i; c0 += 32) {
          int64_t c = c0 + lane;
          bool d = c < i && sel[c] == ti;
          if (__ballot_sync(0xffffffffu, d)) dup = true;
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
          if (i < k) emit(O, out + i, load_slot(slot_at(G, d0, nb, lo + rk)), qkey, i);
        } else {
          // slow exact path: per selected rank, a forward count of valid slots
          for (int l = 0; l < 32 && i0 + l < k; l++) {
            int64_t want = __shfl_sync(0xffffffffu, rk, l);
            int64_t p = lo, seen = 0;
            int64_t b = warp_block_of(G, d0, nb, lo);
            while (p < hi) {
              int64_t cum = __ldg(G.dcum + d0 + b);
              int64_t bend = (b == nb - 1) ? G.nslots[v] : __ldg(G.dcum + d0 + b + 1);
              int64_t cen = min(min(bend, hi), p + 32);
              int64_t pos = p + lane;
              Slot s;
              bool ok = false;
              if (pos < cen) {
                s = load_slot(G.slots + __ldg(G.dbase + d0 + b) + (pos - cum));
                ok = slot_ok(G, s);
              }
              unsigned m = __ballot_sync(0xffffffffu, ok);
              int c = __popc(m);
              if (want < seen + c) {
                int srcl = __fns(m, 0, (int)(want - seen) + 1);
                Slot t2;
                t2.ts = __shfl_sync(0xffffffffu, s.ts, srcl);
                t2.eid = __shfl_sync(0xffffffffu, s.eid, srcl);
                t2.nbr = __shfl_sync(0xffffffffu, s.nbr, srcl);
                if (lane == 0) emit(O, out + i0 + l, t2, qkey, i0 + l);
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
  }
}

template <class F>
gf_status cub_call(F f, cudaStream_t s) {
  size_t bytes = 0;
  GF_CUDA(f((void*)nullptr, bytes));
  Scratch tmp(s);
  GF_TRY(tmp.alloc(bytes));
  GF_CUDA(f(tmp.p, bytes));
  return GF_OK;
}

int64_t grid_warps(int64_t n) {
  int64_t blocks = (n + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
  int64_t cap = (int64_t)num_sms() * 64;  // grid-stride beyond this
  return std::max<int64_t>(1, std::min(blocks, cap));
}

gf_status check_args(int64_t n, int64_t fanout, int policy, int64_t delta) {
  if (n < 0) return fail(GF_EINVAL, "negative query count");
  if (fanout < 1) return fail(GF_EINVAL, "fanout must be >= 1");  // sampling.py:240-241
  if (policy < 0 || policy > 2) return fail(GF_EINVAL, "unknown policy kind");  // sampling.py:38-39
  if (policy == GF_POLICY_TIME_WINDOW && delta <= 0) return fail(GF_EINVAL, "time_window policy requires delta > 0");
  return GF_OK;
}

// one layer: count -> scan -> (host total) -> write
gf_status layer_impl(gf_graph* g, const QueryIn& Q, int64_t* d_offsets, int64_t* d_nbr, int64_t* d_eid, int64_t* d_ts,
                     uint64_t* d_out_keys, int64_t out_cap, int64_t* h_total, cudaStream_t s) {
  *h_total = 0;
  GF_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), s));
  if (Q.n == 0) return GF_OK;
  Scratch sb(s);
  Arena A;
  GF_TRY(sb.alloc((size_t)Q.n * 8 * 4 + 4096));
  A.base = sb.as<char>();
  QueryScratch S{A.take<int64_t>(Q.n), A.take<int64_t>(Q.n), A.take<int64_t>(Q.n)};
  int64_t* counts = A.take<int64_t>(Q.n);
  GraphView G = view_of(g);
  GF_LAUNCH(k_sample_count, grid_warps(Q.n), THREADS, 0, s, G, Q, S, counts);
  cudaEvent_t e0 = g_profile.load(std::memory_order_relaxed) ? prof_start(s) : nullptr;
  GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, counts, d_offsets + 1, (int)Q.n, s); }, s));
  if (e0) prof_stop("cub_scan_offsets", s, e0);
  GF_CUDA(cudaMemcpyAsync(h_total, d_offsets + Q.n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  if (*h_total > out_cap) return fail(GF_ERANGE, "output buffer too small");
  if (*h_total == 0) return GF_OK;
  LayerOut O{d_offsets, d_nbr, d_eid, d_ts, d_out_keys};
  GF_LAUNCH(k_sample_write, grid_warps(Q.n), THREADS, 0, s, G, Q, S, O);
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
  if (n >= ((int64_t)1 << 31)) return fail(GF_EINVAL, "too many queries in one call");
  DeviceGuard dg(g->device);
  QueryIn Q{d_src, d_t_start, d_t_end, d_keys, key_base, n, fanout, policy, delta, seed};
  return layer_impl(g, Q, d_offsets, d_nbr, d_eid, d_ts, d_out_keys, out_cap, h_out_total, (cudaStream_t)stream);
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
    h_totals[h] = 0;
  }
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  const bool need_keys = policy != GF_POLICY_RECENT;
  const int64_t* src = d_roots;
  const int64_t* tend = d_ts;
  int64_t n = n_roots;
  Scratch kbuf[2] = {Scratch(s), Scratch(s)};
  const uint64_t* in_keys = nullptr;
  for (int h = 0; h < n_hops; h++) {
    uint64_t* out_keys = nullptr;
    if (need_keys && h + 1 < n_hops) {
      Scratch& kb = kbuf[h & 1];
      GF_TRY(kb.alloc((size_t)std::max<int64_t>(h_caps[h], 1) * 8));
      out_keys = kb.as<uint64_t>();
    }
    QueryIn Q{src, nullptr, tend, in_keys, root_key_base, n, h_fanouts[h], policy, delta, gf::seed_sequence_2(seed, h)};
    int64_t tot = 0;
    gf_status st = layer_impl(g, Q, d_offsets[h], d_nbr[h], d_eid[h], d_ts_out[h], out_keys, h_caps[h], &tot, s);
    h_totals[h] = tot;
    if (st != GF_OK) return st;
    src = d_nbr[h];
    tend = d_ts_out[h];
    in_keys = out_keys;
    n = tot;
  }
  return GF_OK;
}

}  // extern "C"
