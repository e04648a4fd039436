// gf_sample.cu -- temporal k-hop sampler (K2 window search + selection, K3 CSR output).
//
// Replaces sample_layer / _sample_one / _collect_candidates / _select and the
// sample_khop hop loop (reference sampling.py:145-299).
//
// Timestamps never decrease along a node's block list (storage.py:426-437
// rejects out-of-order edges), so the in-window candidates of a query are one
// contiguous run [lo, hi) of list positions.  Finding hi replaces the
// reference's tail->head block walk with block skipping (sampling.py:157-172):
//   1. the node's 128-byte NodeRec -- if the tail block's tmin is below
//      t_end the boundary is in the tail block (the common case for recent
//      roots), else an interpolation/bisection search over the node's block
//      directory (32-byte entries, one 256-bit load per probe);
//   2. the same search over the block's fence index (32-bit fences every 16
//      slots while every timestamp fits int32, else int64 fences every 32);
//   3. one 16- (or 32-) timestamp window of the dense ts array.
// Selection:
//   recent:     the k newest valid candidates, newest first (sampling.py:188-190) -- bit-exact.
//   uniform/tw: k distinct candidates by Floyd's algorithm on a Philox4x32-10 stream
//               keyed by (hop seed, query key); positions map to slots by the
//               sizing law's closed form (or the directory for irregular lists).
// Output (K3): fast path -- one fused kernel per hop (k_sample_fused: search,
// tile scan with decoupled look-back, selection, cooperative gather/store);
// hop totals stay on the device, so a k-hop call is k launches and one host
// synchronisation.  The unfused count -> scan -> write kernels remain for
// fanout > 16 and for A/B (GF_NO_FUSED).
//
// General path (after deletions): one warp per query, scanning candidate
// validity (valid edge and valid neighbour, sampling.py:178).
#include <cub/cub.cuh>

#include <string.h>

#include <algorithm>
#include <vector>

#include "gf_graph.cuh"

// A/B switches (scripts/build_variant.sh): two measurement-only variants that drop the last hop's
// record loads or its output stores
#ifndef GF_AB_NOGATHER
#define GF_AB_NOGATHER 0
#endif
#ifndef GF_AB_NOSTORE
#define GF_AB_NOSTORE 0
#endif
// measurement only: per-tile phase timestamps of the fused kernel (globaltimer, ns)
#ifndef GF_AB_TRACE
#define GF_AB_TRACE 0
#endif
#if GF_AB_TRACE
constexpr int TRACE_TILES = 1 << 18;
__device__ unsigned long long g_trace[TRACE_TILES][5];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GF_TRACE(tile, i)                                                   \
  do {                                                                      \
    if (threadIdx.x == 0 && (tile) < TRACE_TILES) g_trace[tile][i] = gtimer(); \
  } while (0)
#else
#define GF_TRACE(tile, i) \
  do {                    \
  } while (0)
#endif

using namespace gf;

namespace {

constexpr int THREADS = 256;

struct QueryIn {
  const int64_t* src;
  const int64_t* t_start;  // NULL => TS_MIN
  const int64_t* t_end;
  const uint64_t* keys;    // NULL => key_base + q
  uint64_t key_base;
  int64_t n;               // query count when n_dev == NULL
  const int64_t* n_dev;    // device-resident query count (previous hop's total)
  int64_t fanout;
  int policy;
  int64_t delta;
  uint64_t seed;
};

// per-query state between the count and write passes
struct QState {
  int64_t* lo;
  int64_t* hi;
  int64_t* slot;  // pool index of the slot at list position hi - 1
  int64_t* cum;   // list position of the first slot of that block
  int64_t* d0;    // directory offset
  int64_t* meta;  // block index of hi-1 (low 32) | num_blocks << 32 | irregular << 63
  int64_t* nv;    // candidates the selection runs over
  int64_t* sel;   // general uniform path: positions chosen by rejection (fanout per query), nv = -1 marks it
};

// General-path uniform / time-window selection over a window with deletions: for a
// window of more than GEN_EXACT positions, positions are drawn uniformly (Philox draws REJ_TAG + d)
// and a draw is kept when its candidate is valid (valid edge and valid neighbour, sampling.py:178)
// and new; fanout keeps give a uniform k-subset of the valid candidates.  Only when REJ_MAX draws
// do not yield them does the exact path run (count every valid candidate, Floyd over their ranks).
// The oracle (oracle/gf_oracle.c) makes the same decisions.
constexpr int64_t GEN_EXACT = 64;
constexpr int KREJ = 32;  // the rejection path serves fanouts up to 32
// draw index offset of the rejection draws: Philox block 2^30 + d/2, disjoint from the Floyd draws
// (blocks 0..15); rand64 keys the block with the low 32 bits of d/2, so 2^40 aliased block d/2
constexpr uint64_t REJ_TAG = 1ull << 31;
__host__ __device__ constexpr int64_t rej_max(int64_t fanout) { return 8 * fanout + 32; }

struct LayerOut {
  const int64_t* offsets;
  int64_t* nbr;
  int64_t* eid;
  int64_t* ts;
  uint64_t* keys;  // optional child keys
  int64_t cap;
  int* overflow;
  int last_hop;    // A/B variants only (GF_AB_NOGATHER / GF_AB_NOSTORE act on the last hop)
};

__device__ __forceinline__ int64_t query_count(const QueryIn& Q) { return Q.n_dev ? *Q.n_dev : Q.n; }

__device__ __forceinline__ int64_t t_start_of(const QueryIn& Q, int64_t q, int64_t te) {
  int64_t tsr = Q.t_start ? Q.t_start[q] : GF_TS_MIN;
  if (Q.policy == GF_POLICY_TIME_WINDOW) tsr = (te < GF_TS_MIN + Q.delta) ? GF_TS_MIN : te - Q.delta;  // sampling.py:202-203
  return tsr;
}

__device__ __forceinline__ Slot load_slot(const Slot* p) {
  int64_t w0, w1, w2, w3;
  ld256_stream(p, w0, w1, w2, w3);
  Slot s;
  s.ts = w0;
  s.eid = w1;
  s.nbr = (int32_t)(w2 & 0xffffffff);
  s.owner = (int32_t)(w2 >> 32);
  s.valid = (uint32_t)(w3 & 0xffffffff);
  s.pad = 0;
  return s;
}

// the three output fields only (ts, eid: one 128-bit load; nbr: one 32-bit load from the same sector)
__device__ __forceinline__ Slot load_out3(const Slot* p) {
  Slot s;
  long long a, b;
  int c;
  asm("ld.global.nc.v2.b64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
  asm("ld.global.nc.b32 %0, [%1];" : "=r"(c) : "l"(reinterpret_cast<const char*>(p) + 16));
  s.ts = a;
  s.eid = b;
  s.nbr = c;
  s.owner = 0;
  s.valid = 1;
  s.pad = 0;
  return s;
}

__device__ __forceinline__ void store_out(const LayerOut& O, int64_t at, const Slot& s, uint64_t qkey, int64_t i) {
#if GF_AB_NOSTORE
  if (O.last_hop) {  // measurement only: the last hop's stores dropped (its queries stay valid)
    if ((s.ts ^ s.eid ^ s.nbr) == 0x5a5a5a5a12345ll) *O.overflow = 2;  // keeps the loads live
    return;
  }
#endif
  if (at >= O.cap) {
    *O.overflow = 1;
    return;
  }
  __stcs((long long*)O.nbr + at, (long long)s.nbr);
  __stcs((long long*)O.eid + at, (long long)s.eid);
  __stcs((long long*)O.ts + at, (long long)s.ts);
  if (O.keys) __stcs((long long*)O.keys + at, (long long)child_key(qkey, (uint64_t)i));
}

// 64-bit division out of line: a power-of-two law shifts, and the division's inline expansion at
// every pick site of the unrolled selection loops bloated the kernels past the instruction cache
__device__ __noinline__ int64_t div64_ol(int64_t a, int64_t b) { return a / b; }

// closed-form block index of a list position for regular lists (SizingLaw)
__device__ __forceinline__ int64_t law_block(const SizingLaw& L, int64_t p) {
  if (L.kind == GF_SIZING_FIXED) return L.size_shift >= 0 ? (p >> L.size_shift) : div64_ol(p, L.size);
  if (p >= L.cum_m) return L.m + (L.tau_shift >= 0 ? ((p - L.cum_m) >> L.tau_shift) : div64_ol(p - L.cum_m, L.tau));
  return p == 0 ? 0 : 64 - __clzll(p);
}

// ===================== lane-per-query window search ==========================
// One thread per query: every search step is a single dependent load, but 32
// queries per warp are in flight, and interpolation (timestamps are the
// search keys) keeps the number of steps small.  Directory entries and
// 4-timestamp groups are read with one 256-bit load each.

__device__ __forceinline__ void ld256(const void* p, int64_t& a, int64_t& b, int64_t& c, int64_t& d) {
  asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

// interpolated probe index strictly inside (lo, hi) for key x with known
// neighbour keys tl < x <= th
#ifndef GF_INTERP_STEPS
#define GF_INTERP_STEPS 2
#endif
__device__ __forceinline__ int64_t probe_between(int64_t lo, int64_t hi, int64_t x, int64_t tl, int64_t th, int step) {
  if (step >= GF_INTERP_STEPS || th <= tl) return (lo + hi) >> 1;  // interpolation twice, then bisection
  float f = __fdividef((float)(x - tl), (float)(th - tl));
  int64_t g = lo + 1 + (int64_t)(f * (float)(hi - lo - 1));
  return g <= lo ? lo + 1 : (g >= hi ? hi - 1 : g);
}

// 32-bit run-relative form of probe_between
__device__ __forceinline__ int probe_rel(int lo, int hi, int64_t x, int64_t tl, int64_t th, int step) {
  if (step >= GF_INTERP_STEPS || th <= tl) return (lo + hi) >> 1;
  const float f = __fdividef((float)(x - tl), (float)(th - tl));
  const int g = lo + 1 + __float2int_rz(f * (float)(hi - lo - 1));
  return min(max(g, lo + 1), hi - 1);
}

// Bracketed interpolation search over a sorted int64 run, indices relative to `run`
// (whose absolute index has residue `mis` mod 4).  On entry run[lo] < x <= run[hi], either
// end possibly virtual (outside the run), with known values tl = run[lo], th = run[hi].
// Each probe reads the 32-byte-aligned 4-entry chunk around an interpolated index (one
// 256-bit load).  Within the chunk the predicate "idx <= lo || (idx < hi && v < x)" is a
// prefix of trues, so its popcount k places the boundary directly.  On exit hi = lo + 1 is
// the first index with run[i] >= x.
__device__ __forceinline__ void bracket_search(const int64_t* __restrict__ run, int mis, int& lo, int& hi, int64_t& tl,
                                               int64_t& th, int64_t x) {
  for (int step = 0; hi - lo > 1; step++) {
    const int g0 = ((probe_rel(lo, hi, x, tl, th, step) + mis) & ~3) - mis;
    int64_t v0, v1, v2, v3;
    ld256(run + g0, v0, v1, v2, v3);
    const bool p0 = g0 <= lo || (g0 < hi && v0 < x);
    const bool p1 = g0 + 1 <= lo || (g0 + 1 < hi && v1 < x);
    const bool p2 = g0 + 2 <= lo || (g0 + 2 < hi && v2 < x);
    const bool p3 = g0 + 3 <= lo || (g0 + 3 < hi && v3 < x);
    const int k = (int)p0 + (int)p1 + (int)p2 + (int)p3;
    if (k > 0 && g0 + k - 1 > lo) {
      lo = g0 + k - 1;
      tl = p2 ? (p3 ? v3 : v2) : (p1 ? v1 : v0);  // run[g0 + k - 1]
    }
    if (k < 4 && g0 + k < hi) {
      hi = g0 + k;
      th = p1 ? (p2 ? v3 : v2) : (p0 ? v1 : v0);  // run[g0 + k]
    }
  }
}

// bracket_search over a sorted int32 run (the 32-bit fence): 8 entries per 256-bit chunk
__device__ __forceinline__ int64_t pick32(int64_t w0, int64_t w1, int64_t w2, int64_t w3, int i) {
  const int64_t w = (i & 4) ? ((i & 2) ? w3 : w2) : ((i & 2) ? w1 : w0);
  return (int64_t)(int32_t)((i & 1) ? (uint64_t)w >> 32 : (uint64_t)w);
}

// Callers start with the virtual bracket lo = -1, hi = n (the run length).  Inside the run the values
// ascend and run[lo] < x <= run[hi], so a chunk's count is the entries before the run (virtual, < x)
// plus the run entries < x: one 8-bit compare mask masked to the run, no per-entry bracket tests.
__device__ __forceinline__ void bracket_search32(const int32_t* __restrict__ run, int mis, int& lo, int& hi, int64_t& tl,
                                                 int64_t& th, int64_t x) {
  const int n = hi;
  // every stored timestamp fits int32 here (ts32): v < x is all-true above INT32_MAX, all-false below
  const unsigned all = x > (int64_t)INT32_MAX ? 0xffu : 0u;
  const bool cmp = x > (int64_t)INT32_MIN && x <= (int64_t)INT32_MAX;
  const int32_t x32 = (int32_t)x;
  for (int step = 0; hi - lo > 1; step++) {
    const int g0 = ((probe_rel(lo, hi, x, tl, th, step) + mis) & ~7) - mis;
    int64_t w0, w1, w2, w3;
    ld256(run + g0, w0, w1, w2, w3);
    const int32_t v[8] = {(int32_t)w0, (int32_t)(w0 >> 32), (int32_t)w1, (int32_t)(w1 >> 32),
                          (int32_t)w2, (int32_t)(w2 >> 32), (int32_t)w3, (int32_t)(w3 >> 32)};
    unsigned mv = all;
    if (cmp) {
#pragma unroll
      for (int i = 0; i < 8; i++) mv |= (v[i] < x32) ? (1u << i) : 0u;
    }
    const int neg = min(max(-g0, 0), 8);      // chunk entries before the run
    const int inr = min(max(n - g0, 0), 8);   // chunk entries before the run's end
    const unsigned mr = ((1u << inr) - 1u) & ~((1u << neg) - 1u);
    const int k = neg + __popc(mv & mr);
    if (k > 0 && g0 + k - 1 > lo) {
      lo = g0 + k - 1;
      tl = pick32(w0, w1, w2, w3, k - 1);
    }
    if (k < 8 && g0 + k < hi) {
      hi = g0 + k;
      th = pick32(w0, w1, w2, w3, k);
    }
  }
}

// count of timestamps < x in sts[base, base + size) whose values lie in [t0, t1]
__device__ __forceinline__ int64_t lane_block_lower_bound(const GraphView& GV, int64_t base, int64_t size, int64_t t0,
                                                          int64_t t1, int64_t x) {
  if (x > t1) return size;
#ifndef GF_NO_FENCE
  if (GV.ts32) {
    // 32-bit fences every 32 pool slots (fts32[f] = ts[32 f]; 8 per 256-bit probe) narrow the
    // boundary to [a, b], which lies inside ONE aligned 32-slot group: one 128 B line of sts32
    int64_t a = base, b = base + size, tl = t0 - 1, th = t1 + 1;
    const int64_t f0 = (base + FENCE32 - 1) / FENCE32, f1 = (base + size - 1) / FENCE32;
    if (f1 >= f0) {
      const int nf = (int)(f1 - f0) + 1;
      int flo = -1, fhi = nf;
      int64_t ftl = tl, fth = th;
      bracket_search32(GV.fts32 + f0, (int)(f0 & 7), flo, fhi, ftl, fth, x);
      if (flo >= 0) {
        a = (f0 + flo) * FENCE32 + 1;  // ts[a - 1] = ftl < x
        tl = ftl;
      }
      if (fhi < nf) {
        b = (f0 + fhi) * FENCE32;  // ts[b] = fth >= x
        th = fth;
      }
    }
    if (b <= a) return a - base;
    // inside the window: the same bracketed interpolation over sts32 (8 timestamps per 256-bit
    // probe, usually one probe; a second one hits the line the first brought into L2)
    int lo = -1, hi = (int)(b - a);
    bracket_search32(GV.sts32 + a, (int)(a & 7), lo, hi, tl, th, x);
    return a + hi - base;
  }
#endif
  // bracket relative to base; block sizes are bounded by the sizing law / one ingest batch
  int lo = -1, hi = (int)size;
  int64_t tl = t0 - 1, th = t1 + 1;
#ifndef GF_NO_FENCE
  if (size > FENCE) {
    // the fences f0..f1 (fts[f] = sts[f * FENCE], a 32x smaller array that stays in L2)
    // narrow the bracket to one 32-slot segment first
    const int64_t f0 = (base + FENCE - 1) / FENCE;
    const int nf = (int)((base + size - 1) / FENCE - f0) + 1;
    int flo = -1, fhi = nf;
    int64_t ftl = tl, fth = th;
    bracket_search(GV.fts + f0, (int)(f0 & 3), flo, fhi, ftl, fth, x);
    const int off = (int)(f0 * FENCE - base);  // first fenced slot, relative
    if (flo >= 0) {
      lo = off + flo * FENCE;
      tl = ftl;
    }
    if (fhi < nf) {
      hi = off + fhi * FENCE;
      th = fth;
    }
  }
#endif
  bracket_search(GV.sts + base, (int)(base & 3), lo, hi, tl, th, x);
  return hi;
}

struct LaneNode {
  int64_t d0, ns, nb, first, tcum, tbase, ttmin, tmax, htmin;
  bool valid, irregular;
};

struct LaneBnd {
  int64_t pos, cum, base;  // boundary; block holding pos-1: its first position and slot base
};

// The block holding the last timestamp < x: {first list position, slot base, size, tmin, tmax}.
// none = every block starts at or after x (no position precedes the boundary).
struct LaneBlk {
  int64_t cum, base, size, t0, t1;
  bool none;
};

__device__ __forceinline__ LaneBlk lane_find_block(const GraphView& GV, const LaneNode& N, int64_t x) {
  LaneBlk B;
  B.none = N.htmin >= x;
  if (B.none) return B;
  if (N.ttmin < x) {  // boundary in the tail block
    B.cum = N.tcum;
    B.base = N.tbase;
    B.size = N.ns - N.tcum;
    B.t0 = N.ttmin;
    B.t1 = N.tmax;
    return B;
  }
  // last non-tail block with tmin < x: entries lo < b < hi, tmin[lo] < x <= tmin[hi].
  // Each probe reads entries g and g+1 together, so an exact interpolation ends the search.
  const int64_t* d = GV.dir + N.d0 * DIRW;
  int64_t lo = 0, hi = N.nb - 1, tl = N.htmin, th = N.ttmin;
  int64_t lo_e1 = -1, lo_e2 = 0, lo_e3 = 0, hi_cum = N.tcum;  // cum/base/tmax of lo, cum of hi
  for (int step = 0; hi - lo > 1; step++) {
    const int64_t g = probe_between(lo, hi, x, tl, th, step);
    int64_t e0, e1, e2, e3, n0 = 0, n1 = 0, n2, n3;
    ld256(d + g * DIRW, e0, e1, e2, e3);
    const bool two = g + 1 < hi;
    if (two) ld256(d + (g + 1) * DIRW, n0, n1, n2, n3);
    if (e0 < x) {
      lo = g;
      tl = e0;
      lo_e1 = e1;
      lo_e2 = e2;
      lo_e3 = e3;
      if (two) {
        if (n0 < x) {
          lo = g + 1;
          tl = n0;
          lo_e1 = n1;
          lo_e2 = n2;
          lo_e3 = n3;
        } else {
          hi = g + 1;
          th = n0;
          hi_cum = n1;
        }
      }
    } else {
      hi = g;
      th = e0;
      hi_cum = e1;
    }
  }
  if (lo_e1 < 0) {  // entry lo (= 0) was never probed
    int64_t e0;
    ld256(d + lo * DIRW, e0, lo_e1, lo_e2, lo_e3);
  }
  B.cum = lo_e1;
  B.base = lo_e2;
  B.t0 = tl;
  B.t1 = lo_e3;
  B.size = hi_cum - lo_e1;
  return B;
}

__device__ __forceinline__ LaneBnd lane_list_lower_bound(const GraphView& GV, const LaneNode& N, int64_t x) {
  const LaneBlk B = lane_find_block(GV, N, x);
  if (B.none) return LaneBnd{N.first, 0, 0};
  return LaneBnd{B.cum + lane_block_lower_bound(GV, B.base, B.size, B.t0, B.t1, x), B.cum, B.base};
}

#ifndef GF_COUNT_MINB
#define GF_COUNT_MINB 4  // 64 registers, 32 warps per SM (A/B vs 48 and 40 registers: fastest)
#endif
__global__ void __launch_bounds__(THREADS, GF_COUNT_MINB) k_count_lane(GraphView GV, QueryIn Q, QState S, int64_t* counts, int64_t cap_q) {
  const int64_t n = query_count(Q);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cap_q; q += (int64_t)gridDim.x * blockDim.x) {
    if (q >= n) {
      counts[q] = 0;
      continue;
    }
    const int64_t v = Q.src[q];
    const int64_t te = Q.t_end[q];
    int64_t k = 0;
    if (v >= 0 && v < GV.num_nodes) {
      const int64_t* r = GV.nrec + v * NREC;
      LaneNode N;
      int64_t w2, w3;
      ld256(r, N.d0, N.ns, w2, N.first);
      ld256(r + 4, N.tcum, N.tbase, N.ttmin, N.tmax);
      ld256(r + 8, N.htmin, w3, w3, w3);
      N.nb = w2 & 0xffffffffll;
      N.valid = (w2 & NREC_VALID) != 0;
      N.irregular = (w2 & NREC_IRREG) != 0;
      if (N.valid && N.nb > 0) {  // sampling.py:153-155
        const LaneBnd h = lane_list_lower_bound(GV, N, te);
        const int64_t tsr = t_start_of(Q, q, te);
        const int64_t lo = (tsr == GF_TS_MIN) ? N.first : lane_list_lower_bound(GV, N, tsr).pos;
        if (h.pos > lo) {
          k = min(h.pos - lo, Q.fanout);
          S.lo[q] = lo;
          S.hi[q] = h.pos;
          S.slot[q] = h.base + (h.pos - 1 - h.cum);
          S.cum[q] = h.cum;
          S.d0[q] = N.d0;
          S.meta[q] = (N.nb << 32) | (N.irregular ? (1ll << 62) : 0);
        }
      }
    }
    counts[q] = k;
  }
}

// cum (first list position) of block b for regular lists (SizingLaw)
__device__ __forceinline__ int64_t law_cum(const SizingLaw& L, int64_t b) {
  if (L.kind == GF_SIZING_FIXED) return b * L.size;
  if (b <= L.m) return b == 0 ? 0 : (1ll << (b - 1));
  return L.cum_m + (b - L.m) * L.tau;
}


// per-thread: directory index of the block holding list position p (cum is word 1)
__device__ __forceinline__ int64_t dir_block_of(const GraphView& GV, int64_t d0, int64_t nb, int64_t p) {
  const int64_t* d = GV.dir + d0 * DIRW + 1;
  int64_t lo = 0, hi = nb;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (__ldg(d + m * DIRW) <= p) lo = m + 1;
    else hi = m;
  }
  return lo - 1;
}

__device__ __forceinline__ Slot slot_at_position(const GraphView& GV, bool irregular, int64_t d0, int64_t nb, int64_t p) {
  int64_t b, cum;
  const int64_t* d = GV.dir + d0 * DIRW;
  if (irregular) {
    b = dir_block_of(GV, d0, nb, p);
    cum = __ldg(d + b * DIRW + 1);
  } else {
    b = law_block(GV.law, p);
    cum = law_cum(GV.law, b);
  }
  return load_slot(GV.slots + __ldg(d + b * DIRW + 2) + (p - cum));
}

constexpr int WG = 16;  // lanes per query in the write pass: one output per lane

__global__ void __launch_bounds__(THREADS) k_write_fast(GraphView GV, QueryIn Q, QState S, LayerOut O) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (WG - 1), gbase = lane & WG;
  const unsigned mask = 0xFFFFu << gbase;
  const int64_t n = query_count(Q);
  const int64_t gid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / WG;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / WG;
  for (int64_t q = gid; q < n; q += ngroups) {
    const int64_t out = O.offsets[q];
    const int64_t k = O.offsets[q + 1] - out;
    if (k == 0) continue;
    const int64_t lo = S.lo[q], hi = S.hi[q], nv = hi - lo;
    const uint64_t qkey = Q.keys ? Q.keys[q] : Q.key_base + (uint64_t)q;
    if (Q.policy == GF_POLICY_RECENT || k == nv) {
      // newest first: output r is list position hi-1-r (sampling.py:188-190)
      const int64_t slot_hi = S.slot[q], inblk = hi - S.cum[q];
      for (int64_t r = gl; r < k; r += WG) {
        Slot s;
        if (r < inblk) {
          s = load_slot(GV.slots + slot_hi - r);
        } else {  // crosses into earlier blocks
          const int64_t meta = S.meta[q];
          s = slot_at_position(GV, (meta >> 62) & 1, S.d0[q], meta >> 32 & 0x3fffffff, hi - 1 - r);
        }
        store_out(O, out + r, s, qkey, r);
      }
      continue;
    }
    // uniform / time_window with k < nv: Floyd's algorithm over candidate indices
    const int64_t meta = S.meta[q], d0 = S.d0[q];
    const bool irregular = (meta >> 62) & 1;
    const int64_t nb = meta >> 32 & 0x3fffffff;
    if (k <= WG) {
      int64_t t = 0, sel = -1;
      if (gl < k) {
        // draw i = gl: lanes 2m and 2m+1 evaluate the same Philox block
        uint32_t c[4] = {(uint32_t)(gl >> 1), (uint32_t)qkey, (uint32_t)(qkey >> 32), GF_PHILOX_TAG};
        philox4x32_10(c, (uint32_t)Q.seed, (uint32_t)(Q.seed >> 32));
        uint64_t r = (gl & 1) ? ((uint64_t)c[2] | ((uint64_t)c[3] << 32)) : ((uint64_t)c[0] | ((uint64_t)c[1] << 32));
        t = (int64_t)bounded64(r, (uint64_t)(nv - k + gl + 1));
      }
      for (int i = 0; i < (int)k; i++) {
        int64_t ti = __shfl_sync(mask, t, gbase + i);
        bool dup = (__ballot_sync(mask, gl < i && sel == ti) & mask) != 0;
        if (gl == i) sel = dup ? (nv - k + i) : ti;
      }
      if (gl < k) store_out(O, out + gl, slot_at_position(GV, irregular, d0, nb, lo + sel), qkey, gl);
      continue;
    }
    // large fanout: keep the Floyd set in the output's eid column while drawing
    if (out + k > O.cap) {
      if (gl == 0) *O.overflow = 1;
      continue;
    }
    int64_t* setv = O.eid + out;
    for (int64_t i = 0; i < k; i++) {
      int64_t j = nv - k + i;
      int64_t ti = (int64_t)bounded64(rand64(Q.seed, qkey, (uint64_t)i), (uint64_t)(j + 1));
      bool dup = false;
      for (int64_t c0 = 0; c0 < i; c0 += WG) {
        int64_t c = c0 + gl;
        if (__ballot_sync(mask, c < i && setv[c] == ti) & mask) dup = true;
      }
      __syncwarp(mask);
      if (gl == 0) setv[i] = dup ? j : ti;
      __syncwarp(mask);
    }
    for (int64_t i0 = 0; i0 < k; i0 += WG) {
      int64_t i = i0 + gl;
      int64_t rk = (i < k) ? setv[i] : -1;
      __syncwarp(mask);
      if (i < k) store_out(O, out + i, slot_at_position(GV, irregular, d0, nb, lo + rk), qkey, i);
      __syncwarp(mask);
    }
  }
}

// Write pass for fanout <= KMAX: one lane per query selects its k slots
// (recent: the k newest positions; uniform: Philox draws + Floyd, in
// registers), then the warp moves the 32 queries' outputs cooperatively:
// output e of the warp's contiguous output range is handled by lane e % 32,
// so slot loads have 32 independent addresses in flight and every store
// instruction writes 32 consecutive int64s.
constexpr int KMAX = 16;

__global__ void __launch_bounds__(THREADS) k_write_coop(GraphView GV, QueryIn Q, QState S, LayerOut O) {
  __shared__ uint32_t s_sel[THREADS / 32][32][KMAX];  // pool index of every selected slot
  __shared__ uint8_t s_owner[THREADS / 32][32 * KMAX];
  __shared__ uint64_t s_key[THREADS / 32][32];
  __shared__ int32_t s_pre[THREADS / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n = query_count(Q);
  const int64_t nchunks = (n + 31) / 32;
  for (int64_t chunk = blockIdx.x * (int64_t)(THREADS / 32) + w; chunk < nchunks;
       chunk += (int64_t)gridDim.x * (THREADS / 32)) {
    const int64_t q = chunk * 32 + lane;
    int k = 0;
    int64_t out = 0;
    if (q < n) {
      out = O.offsets[q];
      k = (int)(O.offsets[q + 1] - out);
    }
    if (k > 0) {
      const int64_t lo = S.lo[q], hi = S.hi[q], nv = hi - lo;
      const uint64_t qkey = Q.keys ? Q.keys[q] : Q.key_base + (uint64_t)q;
      s_key[w][lane] = qkey;
      if (Q.policy == GF_POLICY_RECENT || k == nv) {
        // newest first: output r is list position hi-1-r (sampling.py:188-190)
        const int64_t slot_hi = S.slot[q], inblk = hi - S.cum[q];
#pragma unroll
        for (int r = 0; r < KMAX; r++) {
          if (r < k) {
            int64_t sl;
            if (r < inblk) {
              sl = slot_hi - r;
            } else {  // crosses into earlier blocks (short lists)
              const int64_t meta = S.meta[q], d0 = S.d0[q], nb = meta >> 32 & 0x3fffffff;
              const int64_t p = hi - 1 - r;
              const int64_t b = dir_block_of(GV, d0, nb, p);
              const int64_t* e = GV.dir + (d0 + b) * DIRW;
              sl = __ldg(e + 2) + (p - __ldg(e + 1));
            }
            s_sel[w][lane][r] = (uint32_t)sl;
          }
        }
      } else {
        // uniform / time_window (k < nv): Floyd over candidate indices 0..nv-1,
        // draws t_i in [0, nv-k+i] from Philox block i/2 (two draws per block)
        int32_t pick[KMAX];
#pragma unroll
        for (int i = 0; i < KMAX; i += 2) {
          if (i < k) {
            uint32_t c[4] = {(uint32_t)(i >> 1), (uint32_t)qkey, (uint32_t)(qkey >> 32), GF_PHILOX_TAG};
            philox4x32_10(c, (uint32_t)Q.seed, (uint32_t)(Q.seed >> 32));
            int64_t t0 = (int64_t)bounded64((uint64_t)c[0] | ((uint64_t)c[1] << 32), (uint64_t)(nv - k + i + 1));
            bool dup0 = false;
#pragma unroll
            for (int j = 0; j < KMAX; j++) dup0 |= (j < i) && pick[j] == (int32_t)t0;
            pick[i] = dup0 ? (int32_t)(nv - k + i) : (int32_t)t0;
            if (i + 1 < k) {
              int64_t t1 = (int64_t)bounded64((uint64_t)c[2] | ((uint64_t)c[3] << 32), (uint64_t)(nv - k + i + 2));
              bool dup1 = false;
#pragma unroll
              for (int j = 0; j < KMAX; j++) dup1 |= (j < i + 1) && pick[j] == (int32_t)t1;
              pick[i + 1] = dup1 ? (int32_t)(nv - k + i + 1) : (int32_t)t1;
            }
          }
        }
        const int64_t meta = S.meta[q], d0 = S.d0[q];
        const bool irregular = (meta >> 62) & 1;
        const int64_t nb = meta >> 32 & 0x3fffffff;
        const int64_t* dd = GV.dir + d0 * DIRW;
#pragma unroll
        for (int i = 0; i < KMAX; i++) {
          if (i < k) {
            const int64_t p = lo + pick[i];
            int64_t b, cum;
            if (irregular) {
              b = dir_block_of(GV, d0, nb, p);
              cum = __ldg(dd + b * DIRW + 1);
            } else {
              b = law_block(GV.law, p);
              cum = law_cum(GV.law, b);
            }
            s_sel[w][lane][i] = (uint32_t)(__ldg(dd + b * DIRW + 2) + (p - cum));
          }
        }
      }
    }
    // warp scan of the counts: the 32 queries' outputs are one contiguous range
    int incl = k;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int pre = incl - k;
    s_pre[w][lane] = pre;
    for (int i = 0; i < k; i++) s_owner[w][pre + i] = (uint8_t)lane;
    const int64_t out0 = __shfl_sync(0xffffffffu, out, 0);  // outputs of the chunk start at offsets[chunk * 32]
    __syncwarp();
    for (int e = lane; e < total; e += 32) {
      const int j = s_owner[w][e];
      const int i = e - s_pre[w][j];
      const Slot s = load_slot(GV.slots + s_sel[w][j][i]);
      store_out(O, out0 + e, s, s_key[w][j], i);
    }
    __syncwarp();
  }
}

// ===================== fused single-pass layer (fast path) ====================
// k_count_lane + scan + k_write_coop in one kernel: each CTA takes the next
// 256-query tile by ticket (so every lower tile is already resident), runs the
// lane-per-query window search, scans its counts, publishes the tile aggregate,
// selects its slots into shared memory, resolves its output base by decoupled
// look-back over the predecessors' published aggregates, then gathers and
// stores the tile's CSR range.  The per-query search state never leaves
// registers (no QState round trip), offsets are written once, and the
// latency-bound search of one tile overlaps the bandwidth-bound gather of
// others on the same SM.

// status word: flag (bits 63..62) | value; zeroed before each launch
constexpr uint64_t TS_AGG = 1ull << 62, TS_INC = 2ull << 62, TS_VAL = (1ull << 62) - 1;

__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct TileCtl {
  uint64_t* status;             // per tile status word (zeroed before the launch)
  unsigned long long* ticket;   // next tile (zeroed with the status words)
  int64_t* total;               // layer total (written by the tile holding the last query)
};

// pool slot of list position p of an irregular list: the directory's binary search, out of line
__device__ __noinline__ int64_t dir_slot_ol(const int64_t* __restrict__ dd, int64_t nb, int64_t p) {
  int64_t lo = 0, hi = nb;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (__ldg(dd + m * DIRW + 1) <= p) lo = m + 1;
    else hi = m;
  }
  const int64_t b = lo - 1;
  return __ldg(dd + b * DIRW + 2) + (p - __ldg(dd + b * DIRW + 1));
}

// list position -> pool slot for a selected position (regular lists: closed form; else directory)
__device__ __forceinline__ int64_t pool_slot_of64(const GraphView& GV, bool irregular, int64_t d0, int64_t nb, int64_t p) {
  const int64_t* dd = GV.dir + d0 * DIRW;
  int64_t b, cum;
  if (irregular) {
    return dir_slot_ol(dd, nb, p);
  } else {
    b = law_block(GV.law, p);
    cum = law_cum(GV.law, b);
  }
  return __ldg(dd + b * DIRW + 2) + (p - cum);
}
// fused path (pool < 2^32 slots)
__device__ __forceinline__ uint32_t pool_slot_of(const GraphView& GV, bool irregular, int64_t d0, int64_t nb, int64_t p) {
  return (uint32_t)pool_slot_of64(GV, irregular, d0, nb, p);
}
// the same out of line, for the selection loops: inlined at every unrolled pick site the closed-form /
// directory code overflowed the instruction cache (L: the kernel's __grid_constant__ law)
__device__ __noinline__ uint32_t pool_slot_ol(const SizingLaw* __restrict__ L, const int64_t* __restrict__ dir,
                                              int64_t d0, int64_t nb, bool irregular, int64_t p) {
  const int64_t* dd = dir + d0 * DIRW;
  if (irregular) return (uint32_t)dir_slot_ol(dd, nb, p);
  const int64_t b = law_block(*L, p);
  return (uint32_t)(__ldg(dd + b * DIRW + 2) + (p - law_cum(*L, b)));
}

#ifndef GF_FUSED_MINB
#define GF_FUSED_MINB 4
#endif
#ifndef GF_GATHER_UNROLL
#define GF_GATHER_UNROLL 2
#endif

#ifndef GF_GATHER_UNROLL_RECENT
#define GF_GATHER_UNROLL_RECENT 2
#endif

// tile scan of the counts; thread 0 publishes the tile aggregate (tile 0: inclusive prefix)
template <int NW>
__device__ __forceinline__ void tile_publish(int k, int lane, int w, int32_t* s_wsum, const TileCtl& C, int64_t tile,
                                             int& incl, int& wpre, int& agg) {
  incl = k;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[w] = incl;
  __syncthreads();
  wpre = 0;
  agg = 0;
#pragma unroll
  for (int i = 0; i < NW; i++) {
    const int x = s_wsum[i];
    wpre += (i < w) ? x : 0;
    agg += x;
  }
  if (threadIdx.x == 0) st_relaxed(C.status + tile, (tile == 0 ? TS_INC : TS_AGG) | (uint64_t)agg);
}

#ifndef GF_FUSED_THREADS
#define GF_FUSED_THREADS 256
#endif
#ifndef GF_FUSED_THREADS_RECENT
#define GF_FUSED_THREADS_RECENT 128
#endif
// queries per tile = threads per CTA, per policy (A/B: 128 is faster for the latency-bound recent
// hops, 256 for the bandwidth-bound uniform hops)
template <bool EARLY>
constexpr int fused_threads() { return EARLY ? GF_FUSED_THREADS_RECENT : GF_FUSED_THREADS; }

// EARLY: publish the tile aggregate before the in-block window search when every count is
// already known (recent policy: long lists give k = fanout once the boundary block is found)
template <bool EARLY>
#ifndef GF_FUSED_MINB_RECENT
#define GF_FUSED_MINB_RECENT 8  // x 128 threads, 64 registers
#endif
__global__ void __launch_bounds__(fused_threads<EARLY>(),
                                  EARLY ? GF_FUSED_MINB_RECENT : GF_FUSED_MINB * 256 / fused_threads<EARLY>())
    k_sample_fused(const __grid_constant__ GraphView GV, QueryIn Q, LayerOut O, TileCtl C) {
  constexpr int FT = fused_threads<EARLY>();
  constexpr int NW = FT / 32;
  constexpr int GU = EARLY ? GF_GATHER_UNROLL_RECENT : GF_GATHER_UNROLL;  // record loads in flight per lane
  // s_sel[w][lane][(r + lane) % KMAX]: pool slot of a query's r-th pick (rotated so the 32 lanes of a
  // warp writing pick r hit different banks); recent runs inside one block keep only s_hi (slot of
  // position hi-1, all picks are s_hi - r) and skip s_sel
  __shared__ uint32_t s_sel[EARLY ? 1 : NW][32][KMAX];
  // recent: per query the slot of position hi-1 and the positions of the boundary block up to t_end
  // (a pick r < inb is slot s_hi - r); a run crossing into earlier blocks also keeps hi and the
  // node's directory (offset, blocks) to map the older positions
  __shared__ uint32_t s_hi[EARLY ? NW : 1][32];
  __shared__ uint16_t s_inb[EARLY ? NW : 1][32];
  __shared__ int64_t s_xhi[EARLY ? NW : 1][32];
  __shared__ int64_t s_xd0[EARLY ? NW : 1][32];
  __shared__ uint8_t s_owner[NW][32 * KMAX];
  __shared__ uint64_t s_key[NW][32];
  __shared__ int32_t s_pre[NW][32];
  __shared__ int32_t s_wsum[NW];
  __shared__ unsigned s_tile;
  __shared__ int64_t s_base;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = (unsigned)atomicAdd(C.ticket, 1ull);
  __syncthreads();
  const int64_t tile = s_tile;
  if (tile == 0 && threadIdx.x == 0) const_cast<int64_t*>(O.offsets)[0] = 0;
  const int64_t n = query_count(Q);
  if (tile * FT >= n) return;
  const int64_t q = tile * FT + threadIdx.x;
  GF_TRACE(tile, 0);

  // ---- node record + boundary block; the count is often known here already ----
  int k = 0;
  int64_t lo = 0, hi = 0, slot_hi = 0, cum = 0, d0 = 0, nb = 0, te = 0, tsr = GF_TS_MIN;
  bool irregular = false, live = false, known = true;
  uint64_t qkey = 0;
  LaneNode N;
  LaneBlk hb{};
  // window search inside the boundary block
  auto finish = [&]() {
    hi = hb.cum + lane_block_lower_bound(GV, hb.base, hb.size, hb.t0, hb.t1, te);
    lo = (tsr == GF_TS_MIN) ? N.first : lane_list_lower_bound(GV, N, tsr).pos;
    if (hi > lo) {
      k = (int)min(hi - lo, Q.fanout);
      slot_hi = hb.base + (hi - 1 - hb.cum);
      cum = hb.cum;
      d0 = N.d0;
      nb = N.nb;
      irregular = N.irregular;
    } else {
      k = 0;
    }
  };
  if (q < n) {
    const int64_t v = Q.src[q];
    te = Q.t_end[q];
    if (v >= 0 && v < GV.num_nodes) {
      const int64_t* r = GV.nrec + v * NREC;
      int64_t w2, w3;
      ld256(r, N.d0, N.ns, w2, N.first);
      ld256(r + 4, N.tcum, N.tbase, N.ttmin, N.tmax);
      ld256(r + 8, N.htmin, w3, w3, w3);
      N.nb = w2 & 0xffffffffll;
      N.valid = (w2 & NREC_VALID) != 0;
      N.irregular = (w2 & NREC_IRREG) != 0;
      if (N.valid && N.nb > 0) {  // sampling.py:153-155
        tsr = t_start_of(Q, q, te);
        if (EARLY) {
          hb = lane_find_block(GV, N, te);
          live = !hb.none;
          // position hb.cum (tmin < te) is a candidate, so with t_start = TS_MIN there are
          // at least hb.cum + 1 - first of them
          if (live) {
            if (tsr == GF_TS_MIN && hb.cum + 1 - N.first >= Q.fanout) k = (int)Q.fanout;
            else known = false;
          }
        } else {
          const LaneBnd h = lane_list_lower_bound(GV, N, te);
          lo = (tsr == GF_TS_MIN) ? N.first : lane_list_lower_bound(GV, N, tsr).pos;
          if (h.pos > lo) {
            k = (int)min(h.pos - lo, Q.fanout);
            hi = h.pos;
            slot_hi = h.base + (h.pos - 1 - h.cum);
            cum = h.cum;
            d0 = N.d0;
            nb = N.nb;
            irregular = N.irregular;
          }
        }
      }
    }
  }
  int incl = 0, wpre = 0, agg = 0;
  const bool early = EARLY && __syncthreads_and(known);
  if (early) tile_publish<NW>(k, lane, w, s_wsum, C, tile, incl, wpre, agg);

  GF_TRACE(tile, 1);
  if (EARLY && live) finish();
  if (!early) tile_publish<NW>(k, lane, w, s_wsum, C, tile, incl, wpre, agg);

  // ---- selection into shared memory (independent of the output base) ----
  const int pre = incl - k;
  s_pre[w][lane] = pre;
  // the query key feeds only the uniform draws and the child keys, so it is loaded here rather than
  // held in a register through the search
  if ((!EARLY || O.keys) && q < n) qkey = Q.keys ? Q.keys[q] : Q.key_base + (uint64_t)q;
  s_key[w][lane] = qkey;
  for (int i = 0; i < k; i++) s_owner[w][pre + i] = (uint8_t)lane;
  if (k > 0) {
    const int64_t nv = hi - lo;
    if (EARLY || Q.policy == GF_POLICY_RECENT || k == nv) {  // EARLY: launched for recent only
      // newest first: output r is list position hi-1-r (sampling.py:188-190)
      const int64_t inblk = hi - cum;
      if (EARLY) {
        s_hi[EARLY ? w : 0][lane] = (uint32_t)slot_hi;
        s_inb[EARLY ? w : 0][lane] = (uint16_t)min(inblk, (int64_t)KMAX);
        if (k > inblk) {  // the run crosses into earlier blocks (short lists)
          s_xhi[EARLY ? w : 0][lane] = hi;
          s_xd0[EARLY ? w : 0][lane] = d0 | nb << 40 | (irregular ? 1ll << 62 : 0ll);
        }
      } else {
#pragma unroll
        for (int r = 0; r < KMAX; r++) {
          if (r < k)
            s_sel[EARLY ? 0 : w][lane][(r + lane) & (KMAX - 1)] =
                (r < inblk) ? (uint32_t)(slot_hi - r) : pool_slot_ol(&GV.law, GV.dir, d0, nb, irregular, hi - 1 - r);
        }
      }
    } else {
      // uniform / time_window (k < nv): Floyd over candidate indices 0..nv-1,
      // draws t_i in [0, nv-k+i] from Philox block i/2 (two draws per block)
      int32_t pick[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; i += 2) {
        if (i < k) {
          uint32_t c[4] = {(uint32_t)(i >> 1), (uint32_t)qkey, (uint32_t)(qkey >> 32), GF_PHILOX_TAG};
          philox4x32_10(c, (uint32_t)Q.seed, (uint32_t)(Q.seed >> 32));
          const int64_t t0 = (int64_t)bounded64((uint64_t)c[0] | ((uint64_t)c[1] << 32), (uint64_t)(nv - k + i + 1));
          bool dup0 = false;
#pragma unroll
          for (int j = 0; j < KMAX; j++) dup0 |= (j < i) && pick[j] == (int32_t)t0;
          pick[i] = dup0 ? (int32_t)(nv - k + i) : (int32_t)t0;
          if (i + 1 < k) {
            const int64_t t1 = (int64_t)bounded64((uint64_t)c[2] | ((uint64_t)c[3] << 32), (uint64_t)(nv - k + i + 2));
            bool dup1 = false;
#pragma unroll
            for (int j = 0; j < KMAX; j++) dup1 |= (j < i + 1) && pick[j] == (int32_t)t1;
            pick[i + 1] = dup1 ? (int32_t)(nv - k + i + 1) : (int32_t)t1;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < KMAX; i++)
        if (i < k) s_sel[EARLY ? 0 : w][lane][(i + lane) & (KMAX - 1)] = pool_slot_ol(&GV.law, GV.dir, d0, nb, irregular, lo + pick[i]);
    }
  }

  // pool slot of warp output e (query j, pick i)
  auto slot_of = [&](int j, int i) -> uint32_t {
    if (EARLY) {
      const int ww = EARLY ? w : 0;
      if (i < s_inb[ww][j]) return s_hi[ww][j] - (uint32_t)i;
      const int64_t xd = s_xd0[ww][j];
      return pool_slot_of(GV, (xd >> 62) & 1, xd & ((1ll << 40) - 1), (xd >> 40) & ((1ll << 22) - 1), s_xhi[ww][j] - 1 - i);
    }
    return s_sel[EARLY ? 0 : w][j][(i + j) & (KMAX - 1)];
  };
  const int total = __shfl_sync(0xffffffffu, incl, 31);  // the warp's outputs
  // ---- cooperative gather + CSR store of the warp's contiguous range ----
  // recent (contiguous, L2-friendly records): the three output fields with narrow loads; uniform
  // (one random line per record): one 256-bit evict-first load, so the line leaves L2 early (A/B: each
  // choice is the faster one for its policy)
// recent (contiguous, L2-friendly records): the three output fields with narrow loads; uniform
// (one random line per record): one 256-bit evict-first load, so the line leaves L2 early (A/B: each
// choice is the faster one for its policy; SoA copies of the columns made the recent runs cost more
// lines on deep-boundary roots, profiles/README.md)
#if GF_AB_NOGATHER
#define GF_LOAD_OUT(sl) (O.last_hop ? Slot{(int64_t)(sl), 1, 2, 3, 1, 0} : (EARLY ? load_out3(GV.slots + (sl)) : load_slot(GV.slots + (sl))))
#else
#define GF_LOAD_OUT(sl) (EARLY ? load_out3(GV.slots + (sl)) : load_slot(GV.slots + (sl)))
#endif
  // the first gather round is issued before the look-back barrier: its record loads (which need no
  // output base) are in flight while warp 0 resolves the tile's base
  __syncwarp();
  Slot s0[GU];
  int j0[GU];
  int e = lane;
  const bool round0 = e + 32 * (GU - 1) < total;
  if (round0) {
#pragma unroll
    for (int u = 0; u < GU; u++) {
      j0[u] = s_owner[w][e + 32 * u];
      s0[u] = GF_LOAD_OUT(slot_of(j0[u], e + 32 * u - s_pre[w][j0[u]]));
    }
  }

  GF_TRACE(tile, 2);
  // ---- decoupled look-back: output base of this tile ----
  if (w == 0) {
    int64_t excl = 0;
    if (tile > 0) {
      int64_t end = tile - 1;
      while (true) {
        const int64_t idx = end - lane;  // lane 0 = nearest predecessor
        uint64_t st;
        do {
          st = idx >= 0 ? ld_relaxed(C.status + idx) : TS_INC;
        } while (__any_sync(0xffffffffu, (st >> 62) == 0));
        const unsigned inc = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int first = inc ? __ffs(inc) - 1 : 31;
        int64_t v = lane <= first ? (int64_t)(st & TS_VAL) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        end -= 32;
      }
      if (lane == 0) st_relaxed(C.status + tile, TS_INC | (uint64_t)(excl + agg));
    }
    if (lane == 0) s_base = excl;
  }
  __syncthreads();
  const int64_t base = s_base;
  GF_TRACE(tile, 3);
  const int64_t out = base + wpre + pre;
  if (q < n) {
    const_cast<int64_t*>(O.offsets)[q + 1] = out + k;
    if (q == n - 1) *C.total = out + k;
  }

  const int64_t out0 = base + wpre;
  if (round0) {
#pragma unroll
    for (int u = 0; u < GU; u++)
      store_out(O, out0 + e + 32 * u, s0[u], s_key[w][j0[u]], e + 32 * u - s_pre[w][j0[u]]);
    e += 32 * GU;
  }
  for (; e + 32 * (GU - 1) < total; e += 32 * GU) {
    Slot s[GU];
    int j[GU];
#pragma unroll
    for (int u = 0; u < GU; u++) {
      j[u] = s_owner[w][e + 32 * u];
      s[u] = GF_LOAD_OUT(slot_of(j[u], e + 32 * u - s_pre[w][j[u]]));
    }
#pragma unroll
    for (int u = 0; u < GU; u++)
      store_out(O, out0 + e + 32 * u, s[u], s_key[w][j[u]], e + 32 * u - s_pre[w][j[u]]);
  }
  for (; e < total; e += 32) {
    const int jj = s_owner[w][e];
    const int i = e - s_pre[w][jj];
    store_out(O, out0 + e, GF_LOAD_OUT(slot_of(jj, i)), s_key[w][jj], i);
  }
#undef GF_LOAD_OUT
#if GF_AB_TRACE
  if (lane == 0 && tile < TRACE_TILES) atomicMax(&g_trace[tile][4], gtimer());
#endif
}

// ========================== general path (deletions) =========================

__device__ __forceinline__ bool node_ok(const GraphView& G_, int64_t v) {
  return v >= 0 && v < G_.num_nodes && G_.node_valid[v];
}

__device__ __forceinline__ bool slot_ok(const GraphView& G_, const Slot& s) { return s.valid && G_.node_valid[s.nbr]; }

__device__ __forceinline__ int nth_set_bit(unsigned m, int n) {  // 0-based: popcount bisection, no loop
  int pos = 0, c;
  c = __popc(m & 0xffffu);
  if (n >= c) { n -= c; m >>= 16; pos += 16; }
  c = __popc(m & 0xffu);
  if (n >= c) { n -= c; m >>= 8; pos += 8; }
  c = __popc(m & 0xfu);
  if (n >= c) { n -= c; m >>= 4; pos += 4; }
  c = __popc(m & 0x3u);
  if (n >= c) { n -= c; m >>= 2; pos += 2; }
  return pos + ((n >= (int)(m & 1u)) ? 1 : 0);
}

// timestamps < x in the block whose slots are sts[base, base + size)
__device__ __forceinline__ int64_t w_block_lower_bound(const GraphView& GV, int64_t base, int64_t size, int64_t x) {
  const int lane = lane_id();
  int64_t seg_lo = base, seg_hi = base + size;
  if (size > FENCE) {
    int64_t f0 = (base + FENCE - 1) / FENCE, f1 = (base + size - 1) / FENCE;
    int64_t j = warp_lower_bound(GV.fts + f0, 1, f1 - f0 + 1, x);
    if (j == 0) {
      seg_hi = f0 * FENCE;
    } else {
      seg_lo = (f0 + j - 1) * FENCE;
      seg_hi = min(seg_lo + FENCE, base + size);
    }
  }
  int64_t p = seg_lo + lane;
  return seg_lo - base + __popc(__ballot_sync(0xffffffffu, p < seg_hi && __ldg(GV.sts + p) < x));
}

struct WBound {
  int64_t pos, blk;
};

__device__ __forceinline__ WBound w_list_lower_bound(const GraphView& GV, int64_t d0, int64_t nb, int64_t ns_end, int64_t x) {
  int64_t B = warp_lower_bound(GV.dir + d0 * DIRW, DIRW, nb, x);
  if (B == 0) return WBound{__ldg(GV.dir + d0 * DIRW + 1), -1};
  int64_t b = B - 1;
  int64_t cum = __ldg(GV.dir + (d0 + b) * DIRW + 1);
  int64_t size = (b == nb - 1) ? (ns_end - cum) : (__ldg(GV.dir + (d0 + b + 1) * DIRW + 1) - cum);
  return WBound{cum + w_block_lower_bound(GV, __ldg(GV.dir + (d0 + b) * DIRW + 2), size, x), b};
}

__global__ void __launch_bounds__(THREADS) k_count_general(GraphView GV, QueryIn Q, QState S, int64_t* counts, int64_t cap_q) {
  const int lane = threadIdx.x & 31;
  const int64_t n = query_count(Q);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = warp; q < cap_q; q += nwarps) {
    if (q >= n) {
      if (lane == 0) counts[q] = 0;
      continue;
    }
    int64_t v = Q.src[q];
    int64_t lo = 0, hi = 0, nv = 0, k = 0, blk = -1;
    if (node_ok(GV, v) && GV.num_blocks[v] > 0) {
      int64_t nb = GV.num_blocks[v], d0 = GV.dir_off[v], ns = GV.nslots[v];
      int64_t te = Q.t_end[q], tsr = t_start_of(Q, q, te);
      WBound h = w_list_lower_bound(GV, d0, nb, ns, te);
      lo = (tsr == GF_TS_MIN) ? __ldg(GV.dir + d0 * DIRW + 1) : w_list_lower_bound(GV, d0, nb, ns, tsr).pos;
      hi = h.pos > lo ? h.pos : lo;
      blk = h.blk;
      bool rej_done = false;
      if (hi > lo && Q.policy != GF_POLICY_RECENT && hi - lo > GEN_EXACT && Q.fanout <= KREJ) {
        // rejection draws over the window's positions, 32 at a time, accepted in draw order
        const uint64_t qkey = Q.keys ? Q.keys[q] : Q.key_base + (uint64_t)q;
        const int64_t npos = hi - lo, dmax = rej_max(Q.fanout);
        const bool irregular = (GV.nflags[v] & 1) != 0;
        int64_t chosen = -1;  // lane a holds the a-th accepted position
        int acc = 0;
        for (int64_t r0 = 0; r0 < dmax && acc < Q.fanout; r0 += 32) {
          const int64_t d = r0 + lane;
          int64_t p = -1;
          bool ok = false;
          if (d < dmax) {
            p = (int64_t)bounded64(rand64(Q.seed, qkey, REJ_TAG + (uint64_t)d), (uint64_t)npos);
            // deletions leave the block layout on the sizing law until the next allocation
            ok = slot_ok(GV, load_slot(GV.slots + pool_slot_of64(GV, irregular, d0, nb, lo + p)));
          }
          for (int j = 0; j < 32 && acc < Q.fanout; j++) {
            const int64_t pj = __shfl_sync(0xffffffffu, p, j);
            const bool okj = __shfl_sync(0xffffffffu, ok, j);
            const bool dup = __any_sync(0xffffffffu, lane < acc && chosen == pj);
            if (okj && !dup) {
              if (lane == acc) chosen = pj;
              acc++;
            }
          }
        }
        if (acc == Q.fanout) {
          rej_done = true;
          k = acc;
          nv = -1;
          if (lane < acc) S.sel[q * Q.fanout + lane] = lo + chosen;
        }
      }
      if (hi > lo && !rej_done) {
        // valid candidates (sampling.py:178); recent needs at most `fanout`
        int64_t limit = (Q.policy == GF_POLICY_RECENT) ? Q.fanout : INT64_MAX;
        int64_t b = blk, p = hi, cnt = 0;
        while (p > lo && cnt < limit) {
          int64_t cum = __ldg(GV.dir + (d0 + b) * DIRW + 1);
          int64_t cst = max(max(cum, lo), p - 32);
          int64_t pos = p - 1 - lane;
          bool ok = false;
          if (pos >= cst) ok = slot_ok(GV, load_slot(GV.slots + __ldg(GV.dir + (d0 + b) * DIRW + 2) + (pos - cum)));
          cnt += __popc(__ballot_sync(0xffffffffu, ok));
          p = cst;
          if (p == cum) b--;
        }
        nv = cnt < limit ? cnt : limit;
        k = nv < Q.fanout ? nv : Q.fanout;
      }
    }
    if (lane == 0) {
      counts[q] = k;
      S.lo[q] = lo;
      S.hi[q] = hi;
      S.nv[q] = nv;
      S.meta[q] = blk;
    }
  }
}

__global__ void __launch_bounds__(THREADS) k_write_general(GraphView GV, QueryIn Q, QState S, LayerOut O) {
  const int lane = threadIdx.x & 31;
  const int64_t n = query_count(Q);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = warp; q < n; q += nwarps) {
    const int64_t out = O.offsets[q];
    const int64_t k = O.offsets[q + 1] - out;
    if (k == 0) continue;
    int64_t v = Q.src[q];
    int64_t d0 = GV.dir_off[v], nb = GV.num_blocks[v];
    uint64_t qkey = Q.keys ? Q.keys[q] : Q.key_base + (uint64_t)q;
    const int64_t lo = S.lo[q], hi = S.hi[q], nv = S.nv[q];
    if (nv == -1) {  // positions chosen by the rejection draws of the count pass
      const bool irregular = (GV.nflags[v] & 1) != 0;
      for (int64_t i = lane; i < k; i += 32)
        store_out(O, out + i, load_slot(GV.slots + pool_slot_of64(GV, irregular, d0, nb, S.sel[q * Q.fanout + i])), qkey, i);
      continue;
    }
    if (Q.policy == GF_POLICY_RECENT || k == nv) {
      const unsigned lt = (1u << lane) - 1u;
      int64_t b = S.meta[q], p = hi, done = 0;
      while (done < k && p > lo) {
        int64_t cum = __ldg(GV.dir + (d0 + b) * DIRW + 1);
        int64_t cst = max(max(cum, lo), p - 32);
        int64_t pos = p - 1 - lane;
        bool ok = false;
        Slot s;
        if (pos >= cst) {
          s = load_slot(GV.slots + __ldg(GV.dir + (d0 + b) * DIRW + 2) + (pos - cum));
          ok = slot_ok(GV, s);
        }
        unsigned m = __ballot_sync(0xffffffffu, ok);
        int64_t r = done + __popc(m & lt);
        if (ok && r < k) store_out(O, out + r, s, qkey, r);
        done += __popc(m);
        p = cst;
        if (p == cum) b--;
      }
      continue;
    }
    // Floyd's k-of-nv over the chronological valid ranks, then rank -> position scans
    if (out + k > O.cap) {
      if (lane == 0) *O.overflow = 1;
      continue;
    }
    int64_t* setv = O.eid + out;
    for (int64_t i = 0; i < k; i++) {
      int64_t j = nv - k + i;
      int64_t ti = (int64_t)bounded64(rand64(Q.seed, qkey, (uint64_t)i), (uint64_t)(j + 1));
      bool dup = false;
      for (int64_t c0 = 0; c0 < i; c0 += 32) {
        int64_t c = c0 + lane;
        if (__ballot_sync(0xffffffffu, c < i && setv[c] == ti)) dup = true;
      }
      __syncwarp();
      if (lane == 0) setv[i] = dup ? j : ti;
      __syncwarp();
    }
    // one forward pass over [lo, hi): a selected chronological valid rank r is
    // replaced by ~position (negative, so it cannot match again) when reached
    int64_t b = dir_block_of(GV, d0, nb, lo);
    int64_t p = lo, rank0 = 0;
    while (p < hi) {
      int64_t cum = __ldg(GV.dir + (d0 + b) * DIRW + 1);
      int64_t bend = (b == nb - 1) ? GV.nslots[v] : __ldg(GV.dir + (d0 + b + 1) * DIRW + 1);
      int64_t cen = min(min(bend, hi), p + 32);
      int64_t pos = p + lane;
      bool ok = pos < cen && slot_ok(GV, load_slot(GV.slots + __ldg(GV.dir + (d0 + b) * DIRW + 2) + (pos - cum)));
      unsigned m = __ballot_sync(0xffffffffu, ok);
      int c = __popc(m);
      for (int64_t i0 = 0; i0 < k; i0 += 32) {
        int64_t i = i0 + lane;
        int64_t want = (i < k) ? setv[i] : -1;
        if (want >= rank0 && want < rank0 + c) setv[i] = ~(p + nth_set_bit(m, (int)(want - rank0)));
      }
      __syncwarp();
      rank0 += c;
      p = cen;
      if (p == bend) b++;
    }
    for (int64_t i = lane; i < k; i += 32) {
      int64_t ps = ~setv[i];
      int64_t bb = dir_block_of(GV, d0, nb, ps);
      store_out(O, out + i, load_slot(GV.slots + __ldg(GV.dir + (d0 + bb) * DIRW + 2) + (ps - __ldg(GV.dir + (d0 + bb) * DIRW + 1))), qkey, i);
    }
  }
}

// ===================== fused path after deletions (lane per query) ===================
// The general path's decisions (k_count_general / k_write_general, oracle/gf_oracle.c) in the fused
// kernel's shape: the window search of the fast path (deletions are soft, so the list layout and
// its timestamps are unchanged), then a per-lane selection that reads candidate validity
// (valid edge and valid neighbour, sampling.py:178) from the 1-bit-per-slot candidate bitmap:
//   recent             newest first, up to fanout valid, scanning back at most DEL_SCAN positions;
//   uniform / window   more than GEN_EXACT positions: the fast path's Floyd positions, the valid
//                      ones kept; then rejection draws (REJ_TAG + d), 4 in flight, kept in draw
//                      order when valid and new, up to rej_max draws;
//                      at most GEN_EXACT positions: a validity mask of the window, then newest
//                      first (every valid candidate fits) or Floyd over the valid ranks.
// A query a lane cannot finish within those bounds (a recent run past DEL_SCAN, rejection draws
// exhausted) is taken over by its whole warp, 32 positions per step, as the general kernels do.
// Selected pool slots go to the per-query pick array; tile scan, decoupled look-back and the
// cooperative gather/store are those of k_sample_fused.
#ifndef GF_DEL_THREADS
#define GF_DEL_THREADS 512  // A/B: 128 / 256-query tiles 1.3x / 1.12x slower uniform selection
#endif
#ifndef GF_DEL_MINB
#define GF_DEL_MINB 2  // 64 registers (A/B at 256 threads: 2 and 3 CTAs per SM 1.4x / 1.15x slower than 4)
#endif

constexpr int DEL_SCAN = 64;
#if GF_DEL_STATS
__device__ unsigned long long g_del_stats[8];  // A/B instrumentation only (GF_DEL_STATS builds)
#define DEL_STAT(i, v) atomicAdd(&g_del_stats[i], (unsigned long long)(v))
#else
#define DEL_STAT(i, v) ((void)0)
#endif

// Floyd's k distinct indices of [0, nv) (k < nv, k <= KMAX), exactly as k_sample_fused draws them:
// t_i in [0, nv-k+i] from Philox block i/2 keyed by (seed, key) (two draws per block, = rand64),
// a duplicate replaced by nv-k+i
__device__ __forceinline__ void floyd_positions(uint64_t seed, uint64_t qkey, int64_t nv, int k, int32_t (&pick)[KMAX]) {
#pragma unroll
  for (int i = 0; i < KMAX; i += 2) {
    if (i < k) {
      uint32_t c[4] = {(uint32_t)(i >> 1), (uint32_t)qkey, (uint32_t)(qkey >> 32), GF_PHILOX_TAG};
      philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
      const int64_t t0 = (int64_t)bounded64((uint64_t)c[0] | ((uint64_t)c[1] << 32), (uint64_t)(nv - k + i + 1));
      bool dup0 = false;
#pragma unroll
      for (int j = 0; j < KMAX; j++) dup0 |= (j < i) && pick[j] == (int32_t)t0;
      pick[i] = dup0 ? (int32_t)(nv - k + i) : (int32_t)t0;
      if (i + 1 < k) {
        const int64_t t1 = (int64_t)bounded64((uint64_t)c[2] | ((uint64_t)c[3] << 32), (uint64_t)(nv - k + i + 2));
        bool dup1 = false;
#pragma unroll
        for (int j = 0; j < KMAX; j++) dup1 |= (j < i + 1) && pick[j] == (int32_t)t1;
        pick[i + 1] = dup1 ? (int32_t)(nv - k + i + 1) : (int32_t)t1;
      }
    }
  }
}

// rand64 as one out-of-line copy of Philox4x32-10 for the post-deletion kernels: their ~20 draw sites
// inlined made the selection kernel larger than the instruction cache
__device__ __noinline__ uint64_t rand64_ol(uint64_t seed, uint64_t qkey, uint64_t d) { return rand64(seed, qkey, d); }

// Philox block `blk` of the stream keyed by (seed, key), out of line: draws 2 blk and 2 blk + 1
__device__ __noinline__ uint4 philox_block_ol(uint64_t seed, uint64_t qkey, uint32_t blk) {
  uint32_t c[4] = {blk, (uint32_t)qkey, (uint32_t)(qkey >> 32), GF_PHILOX_TAG};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  return make_uint4(c[0], c[1], c[2], c[3]);
}

// floyd_positions with the out-of-line Philox, two draws per block (the same values)
__device__ __forceinline__ void floyd_positions_ol(uint64_t seed, uint64_t qkey, int64_t nv, int k, int32_t (&pick)[KMAX]) {
#pragma unroll
  for (int i = 0; i < KMAX; i += 2) {
    if (i < k) {
      const uint4 c = philox_block_ol(seed, qkey, (uint32_t)(i >> 1));
      const int64_t t0 = (int64_t)bounded64((uint64_t)c.x | ((uint64_t)c.y << 32), (uint64_t)(nv - k + i + 1));
      bool dup0 = false;
#pragma unroll
      for (int j = 0; j < KMAX; j++) dup0 |= (j < i) && pick[j] == (int32_t)t0;
      pick[i] = dup0 ? (int32_t)(nv - k + i) : (int32_t)t0;
      if (i + 1 < k) {
        const int64_t t1 = (int64_t)bounded64((uint64_t)c.z | ((uint64_t)c.w << 32), (uint64_t)(nv - k + i + 2));
        bool dup1 = false;
#pragma unroll
        for (int j = 0; j < KMAX; j++) dup1 |= (j < i + 1) && pick[j] == (int32_t)t1;
        pick[i + 1] = dup1 ? (int32_t)(nv - k + i + 1) : (int32_t)t1;
      }
    }
  }
}

// pool slot sl is a candidate (valid edge, valid neighbour): one bit of the 1-bit-per-slot bitmap the
// deletions maintain (gf_graph.cuh okbits), L2-resident, instead of the slot's own record
__device__ __forceinline__ bool cand_ok(const GraphView& GV, uint32_t sl) {
#if GF_AB_DEL_NOBITS
  return sl != 0xffffffffu;  // A/B timing only: every candidate valid, no bitmap read
#else
  return (__ldg(GV.okbits + (sl >> 5)) >> (sl & 31)) & 1u;
#endif
}

__device__ __forceinline__ int nth_set_bit64(uint64_t m, int r) {  // 0-based position of the r-th set bit
  const unsigned lo = (unsigned)m;
  const int c = __popc(lo);
  return r < c ? nth_set_bit(lo, r) : 32 + nth_set_bit((unsigned)(m >> 32), r - c);
}

// a query's window, as the lane found it: positions [lo, hi); positions >= cum lie in the boundary
// block (slot of hi-1 = slot_hi), earlier ones are mapped through the sizing law or the directory
struct DelWin {
  int64_t lo, hi, cum, slot_hi, d0, nb;
  bool irregular;
};
__device__ __forceinline__ uint32_t del_slot(const GraphView& GV, const DelWin& W, int64_t p) {
  return p >= W.cum ? (uint32_t)(W.slot_hi - (W.hi - 1 - p)) : pool_slot_ol(&GV.law, GV.dir, W.d0, W.nb, W.irregular, p);
}

// bits [s, s + len) of the candidate bitmap (len <= 64; the bitmap is padded past its end)
__device__ __forceinline__ uint64_t run_bits(const GraphView& GV, int64_t s, int len) {
  const int64_t w = s >> 5;
  const int sh = (int)(s & 31);
  const uint64_t a = (uint64_t)__ldg(GV.okbits + w) | ((uint64_t)__ldg(GV.okbits + w + 1) << 32);
  const uint64_t b = (len + sh > 64) ? (uint64_t)__ldg(GV.okbits + w + 2) : 0;
  const uint64_t v = (a >> sh) | (sh ? (b << (64 - sh)) : 0);
  return len >= 64 ? v : (v & ((1ull << len) - 1));
}

// candidate mask of a window of at most 64 positions, bit i = position lo + i: the boundary block's
// part is one contiguous run of slots; each earlier block's run comes from its directory entry
__device__ __forceinline__ uint64_t window_mask(const GraphView& GV, const DelWin& W) {
  const int64_t p0 = max(W.lo, W.cum);
  uint64_t m = run_bits(GV, W.slot_hi - (W.hi - 1 - p0), (int)(W.hi - p0)) << (p0 - W.lo);
  if (W.lo < W.cum) {
    const int64_t* d = GV.dir + W.d0 * DIRW;
    const int64_t b0 = W.irregular ? dir_block_of(GV, W.d0, W.nb, W.lo) : law_block(GV.law, W.lo);
    const int64_t b1 = W.irregular ? dir_block_of(GV, W.d0, W.nb, W.cum - 1) : law_block(GV.law, W.cum - 1);
#pragma unroll 4
    for (int64_t b = b0; b <= b1; b++) {
      const int64_t cb = W.irregular ? __ldg(d + b * DIRW + 1) : law_cum(GV.law, b);
      const int64_t ce = (b == b1) ? W.cum : (W.irregular ? __ldg(d + (b + 1) * DIRW + 1) : law_cum(GV.law, b + 1));
      const int64_t ps = max(W.lo, cb);
      m |= run_bits(GV, __ldg(d + b * DIRW + 2) + (ps - cb), (int)(ce - ps)) << (ps - W.lo);
    }
  }
  return m;
}

// the whole warp selects for one query (uniform after failed draws / recent past DEL_SCAN): the
// general kernels' algorithm; picks go to sel[(i + owner) % KMAX]; returns the count
template <bool RECENT>
__device__ __forceinline__ int warp_select_general(const GraphView& GV, const QueryIn& Q, const DelWin& W, uint64_t qkey,
                                   uint32_t* sel, int owner) {
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  auto put = [&](int i, uint32_t sl) { sel[(i + owner) & (KMAX - 1)] = sl; };
  auto ok_at = [&](int64_t p, uint32_t& sl) {
    sl = del_slot(GV, W, p);
    return cand_ok(GV, sl);
  };
  constexpr bool recent = RECENT;
  int64_t nv = 0;
  if (!recent) {  // every valid candidate counts
    for (int64_t p0 = W.lo; p0 < W.hi; p0 += 32) {
      const int64_t p = p0 + lane;
      uint32_t sl;
      nv += __popc(__ballot_sync(0xffffffffu, p < W.hi && ok_at(p, sl)));
    }
  }
  const int kmax = (int)min((int64_t)Q.fanout, recent ? (int64_t)Q.fanout : nv);
  if (recent || kmax == nv) {  // newest first
    int done = 0;
    for (int64_t p0 = W.hi - 1; p0 >= W.lo && done < kmax; p0 -= 32) {
      const int64_t p = p0 - lane;
      uint32_t sl = 0;
      const bool ok = p >= W.lo && ok_at(p, sl);
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      const int r = done + __popc(m & lt);
      if (ok && r < kmax) put(r, sl);
      done += __popc(m);
    }
    __syncwarp();
    return min(done, kmax);
  }
  // Floyd's k-of-nv over the chronological valid ranks (rand64(seed, key, i)), lane i keeps rank i
  int64_t want = -1;
  for (int i = 0; i < kmax; i++) {
    const int64_t j = nv - kmax + i;
    const int64_t ti = (int64_t)bounded64(rand64_ol(Q.seed, qkey, (uint64_t)i), (uint64_t)(j + 1));
    const bool dup = __any_sync(0xffffffffu, lane < i && want == ti);
    if (lane == i) want = dup ? j : ti;
  }
  int64_t rank0 = 0;
  for (int64_t p0 = W.lo; p0 < W.hi; p0 += 32) {
    const int64_t p = p0 + lane;
    uint32_t sl;
    const unsigned m = __ballot_sync(0xffffffffu, p < W.hi && ok_at(p, sl));
    const int c = __popc(m);
    if (lane < kmax && want >= rank0 && want < rank0 + c) put(lane, del_slot(GV, W, p0 + nth_set_bit(m, (int)(want - rank0))));
    rank0 += c;
  }
  __syncwarp();
  return kmax;
}

// SPLIT (uniform / time-window): the selection ends the kernel -- counts[q] and the picks
// picks[i * cap_q + q] (pick-major: a warp's stores of pick i are one line) go to HBM, a scan gives the
// offsets and k_gather_picks writes the layer.  The
// selection's validity reads make tile times uneven, and in the fused shape every later tile's
// look-back waits on them; recent selections are short and stay fused.
template <bool SPLIT>
__global__ void __launch_bounds__(GF_DEL_THREADS, GF_DEL_MINB)
    k_sample_fused_del(const __grid_constant__ GraphView GV, QueryIn Q, LayerOut O, TileCtl C, int64_t* counts,
                       uint32_t* picks, int64_t cap_q) {
  constexpr int FT = GF_DEL_THREADS;
  constexpr int NW = FT / 32;
  __shared__ uint32_t s_sel[NW][32][KMAX];
  __shared__ uint8_t s_owner[NW][32 * KMAX];
  __shared__ uint64_t s_key[NW][32];
  __shared__ int32_t s_pre[NW][32];
  __shared__ int32_t s_wsum[NW];
  __shared__ unsigned s_tile;
  __shared__ int64_t s_base;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t tile = blockIdx.x;
  if (!SPLIT) {
    if (threadIdx.x == 0) s_tile = (unsigned)atomicAdd(C.ticket, 1ull);
    __syncthreads();
    tile = s_tile;
    if (tile == 0 && threadIdx.x == 0) const_cast<int64_t*>(O.offsets)[0] = 0;
  }
  const int64_t n = query_count(Q);
  if (SPLIT) {  // the scan runs over cap_q counts
    const int64_t qq = tile * FT + threadIdx.x;
    if (qq >= n && qq < cap_q) counts[qq] = 0;
  }
  if (tile * FT >= n) return;
  const int64_t q = tile * FT + threadIdx.x;

  // ---- window search (as the fast path) ----
  DelWin W{0, 0, 0, 0, 0, 0, false};
  uint64_t qkey = 0;
  if (q < n) {
    const int64_t v = Q.src[q];
    const int64_t te = Q.t_end[q];
    qkey = Q.keys ? Q.keys[q] : Q.key_base + (uint64_t)q;
    if (v >= 0 && v < GV.num_nodes) {
      const int64_t* r = GV.nrec + v * NREC;
      LaneNode N;
      int64_t w2, w3;
      ld256(r, N.d0, N.ns, w2, N.first);
      ld256(r + 4, N.tcum, N.tbase, N.ttmin, N.tmax);
      ld256(r + 8, N.htmin, w3, w3, w3);
      N.nb = w2 & 0xffffffffll;
      N.valid = (w2 & NREC_VALID) != 0;  // cleared by delete_node (sampling.py:153-155)
      N.irregular = (w2 & NREC_IRREG) != 0;
      if (N.valid && N.nb > 0) {
        const int64_t tsr = t_start_of(Q, q, te);
        const LaneBnd h = lane_list_lower_bound(GV, N, te);
        const int64_t lo = (tsr == GF_TS_MIN) ? N.first : lane_list_lower_bound(GV, N, tsr).pos;
        if (h.pos > lo) W = DelWin{lo, h.pos, h.cum, h.base + (h.pos - 1 - h.cum), N.d0, N.nb, N.irregular};
      }
    }
  }

  // ---- selection: validity-checked picks into s_sel ----
  uint32_t* sel = &s_sel[w][lane][0];
  int k = 0;
  bool hard = false;
  const int fan = (int)Q.fanout;
  if (W.hi > W.lo) {
    const int64_t npos = W.hi - W.lo;
    // each instantiation carries only its policy's branches (the host launches SPLIT for uniform /
    // time-window and the fused form for recent): one kernel with all of them ran out of the
    // instruction cache (half of its warp stalls were no-instruction)
    if (!SPLIT) {
      // the newest DEL_SCAN positions as one candidate mask; newest first
      DelWin WS = W;
      WS.lo = max(W.lo, W.hi - DEL_SCAN);
      uint64_t mm = window_mask(GV, WS);
      const int64_t stop = WS.lo;
      while (mm && k < fan) {
        const int b = 63 - __clzll(mm);
        mm &= ~(1ull << b);
        sel[(k++ + lane) & (KMAX - 1)] = del_slot(GV, W, stop + b);
      }
      hard = k < fan && stop > W.lo;  // valid candidates may remain below the lane's bound
    } else if (npos > GEN_EXACT) {  // SPLIT
      // Floyd first: the fast path's k distinct positions (the same Philox draws); its candidates are
      // kept (in draw order) -- all of them for every query no deletion touches, which then gets
      // its pre-deletion sample.  Kept Floyd picks are a uniform subset of the valid candidates of
      // a uniform size, so topping them up with uniform new valid draws leaves a uniform k-subset.
      {
        int32_t pick[KMAX];
        floyd_positions_ol(Q.seed, qkey, npos, fan, pick);
        uint32_t sl[KMAX];
#pragma unroll
        for (int i = 0; i < KMAX; i++)
          if (i < fan) sl[i] = del_slot(GV, W, W.lo + pick[i]);
        unsigned okm = 0;  // every bit load in flight together
#pragma unroll
        for (int i = 0; i < KMAX; i++)
          if (i < fan && cand_ok(GV, sl[i])) okm |= 1u << i;
#pragma unroll
        for (int i = 0; i < KMAX; i++)
          if ((okm >> i) & 1) sel[(k++ + lane) & (KMAX - 1)] = sl[i];
        DEL_STAT(4, k < fan ? 1 : 0);
      }
      // then rejection draws over positions (fanout <= KMAX <= KREJ), 4 in flight, kept when valid and new
      const int64_t dmax = rej_max(Q.fanout);
      for (int64_t d = 0; k < fan && d < dmax; d += 4) {
        uint32_t sl[4];
        bool ok[4];
        // draws REJ_TAG + d .. + 3: two Philox blocks (d is even, REJ_TAG too)
        const uint32_t blk = (uint32_t)((REJ_TAG + (uint64_t)d) >> 1);
        const uint4 ca = philox_block_ol(Q.seed, qkey, blk), cb = philox_block_ol(Q.seed, qkey, blk + 1);
        const uint64_t r4[4] = {(uint64_t)ca.x | ((uint64_t)ca.y << 32), (uint64_t)ca.z | ((uint64_t)ca.w << 32),
                                (uint64_t)cb.x | ((uint64_t)cb.y << 32), (uint64_t)cb.z | ((uint64_t)cb.w << 32)};
#pragma unroll
        for (int u = 0; u < 4; u++) {
          ok[u] = false;
          if (d + u < dmax) {
            const int64_t p = W.lo + (int64_t)bounded64(r4[u], (uint64_t)npos);
            sl[u] = del_slot(GV, W, p);
            ok[u] = cand_ok(GV, sl[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          if (ok[u] && k < fan) {
            bool dup = false;
            for (int j = 0; j < k; j++) dup |= sel[(j + lane) & (KMAX - 1)] == sl[u];
            if (!dup) sel[(k++ + lane) & (KMAX - 1)] = sl[u];
          }
        }
      }
      if (k < fan) {  // draws exhausted: the exact path, by the warp
        hard = true;
        k = 0;
      }
    } else {  // exact over at most GEN_EXACT positions: validity mask, bit i = position lo + i
      const uint64_t m = window_mask(GV, W);
      const int nv = __popcll(m);
      k = min(nv, fan);
      if (k == nv) {  // newest first
        uint64_t mm = m;
        for (int i = 0; i < k; i++) {
          const int b = 63 - __clzll(mm);
          mm &= ~(1ull << b);
          sel[(i + lane) & (KMAX - 1)] = del_slot(GV, W, W.lo + b);
        }
      } else {  // Floyd's k-of-nv over the chronological valid ranks (draws rand64 i)
        int32_t t[KMAX];
        floyd_positions_ol(Q.seed, qkey, nv, k, t);
#pragma unroll
        for (int i = 0; i < KMAX; i++)
          if (i < k) sel[(i + lane) & (KMAX - 1)] = del_slot(GV, W, W.lo + nth_set_bit64(m, t[i]));
      }
    }
  }
  DEL_STAT(0, 1);
  DEL_STAT(1, W.hi > W.lo && W.hi - W.lo <= GEN_EXACT ? 1 : 0);
  DEL_STAT(2, hard ? 1 : 0);
  DEL_STAT(3, hard ? W.hi - W.lo : 0);
  // queries the lanes could not finish: their warp takes them one at a time
  for (unsigned hm = __ballot_sync(0xffffffffu, hard); hm; hm &= hm - 1) {
    const int L = __ffs(hm) - 1;
    DelWin WL;
    WL.lo = __shfl_sync(0xffffffffu, W.lo, L);
    WL.hi = __shfl_sync(0xffffffffu, W.hi, L);
    WL.cum = __shfl_sync(0xffffffffu, W.cum, L);
    WL.slot_hi = __shfl_sync(0xffffffffu, W.slot_hi, L);
    WL.d0 = __shfl_sync(0xffffffffu, W.d0, L);
    WL.nb = __shfl_sync(0xffffffffu, W.nb, L);
    WL.irregular = __shfl_sync(0xffffffffu, (int)W.irregular, L) != 0;
    const uint64_t kl = __shfl_sync(0xffffffffu, qkey, L);
    const int kk = warp_select_general<!SPLIT>(GV, Q, WL, kl, &s_sel[w][L][0], L);
    if (lane == L) k = kk;
  }

  if (SPLIT) {
    __syncwarp();
    if (q < n) {
      counts[q] = k;
      for (int i = 0; i < k; i++) picks[i * cap_q + q] = sel[(i + lane) & (KMAX - 1)];
    }
    return;
  }

  // ---- tile scan, owners, look-back, gather/store (k_sample_fused) ----
  int incl = 0, wpre = 0, agg = 0;
  tile_publish<NW>(k, lane, w, s_wsum, C, tile, incl, wpre, agg);
  const int pre = incl - k;
  s_pre[w][lane] = pre;
  s_key[w][lane] = qkey;
  for (int i = 0; i < k; i++) s_owner[w][pre + i] = (uint8_t)lane;
  __syncwarp();
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  auto slot_e = [&](int j, int i) { return s_sel[w][j][(i + j) & (KMAX - 1)]; };
  // the first gather round is issued before the look-back (its loads need no output base)
  constexpr int GU = GF_GATHER_UNROLL;
  Slot s0[GU];
  int j0[GU];
  int e = lane;
  const bool round0 = e + 32 * (GU - 1) < total;
  if (round0) {
#pragma unroll
    for (int u = 0; u < GU; u++) {
      j0[u] = s_owner[w][e + 32 * u];
      s0[u] = load_slot(GV.slots + slot_e(j0[u], e + 32 * u - s_pre[w][j0[u]]));
    }
  }
  if (w == 0) {
    int64_t excl = 0;
    if (tile > 0) {
      int64_t end = tile - 1;
      while (true) {
        const int64_t idx = end - lane;
        uint64_t st;
        do {
          st = idx >= 0 ? ld_relaxed(C.status + idx) : TS_INC;
        } while (__any_sync(0xffffffffu, (st >> 62) == 0));
        const unsigned inc = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int first = inc ? __ffs(inc) - 1 : 31;
        int64_t v = lane <= first ? (int64_t)(st & TS_VAL) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        end -= 32;
      }
      if (lane == 0) st_relaxed(C.status + tile, TS_INC | (uint64_t)(excl + agg));
    }
    if (lane == 0) s_base = excl;
  }
  __syncthreads();
  const int64_t base = s_base;
  const int64_t out = base + wpre + pre;
  if (q < n) {
    const_cast<int64_t*>(O.offsets)[q + 1] = out + k;
    if (q == n - 1) *C.total = out + k;
  }
  const int64_t out0 = base + wpre;
  if (round0) {
#pragma unroll
    for (int u = 0; u < GU; u++) store_out(O, out0 + e + 32 * u, s0[u], s_key[w][j0[u]], e + 32 * u - s_pre[w][j0[u]]);
    e += 32 * GU;
  }
  for (; e + 32 * (GU - 1) < total; e += 32 * GU) {
    Slot sv[GU];
    int jv[GU];
#pragma unroll
    for (int u = 0; u < GU; u++) {
      jv[u] = s_owner[w][e + 32 * u];
      sv[u] = load_slot(GV.slots + slot_e(jv[u], e + 32 * u - s_pre[w][jv[u]]));
    }
#pragma unroll
    for (int u = 0; u < GU; u++) store_out(O, out0 + e + 32 * u, sv[u], s_key[w][jv[u]], e + 32 * u - s_pre[w][jv[u]]);
  }
  for (; e < total; e += 32) {
    const int j = s_owner[w][e];
    const int i = e - s_pre[w][j];
    store_out(O, out0 + e, load_slot(GV.slots + slot_e(j, i)), s_key[w][j], i);
  }
}

// The layer of a split post-deletion selection: a warp per 32 consecutive queries owns their
// contiguous output range and moves it with coalesced stores (as k_sample_fused's gather/store)
__global__ void __launch_bounds__(256) k_gather_picks(GraphView GV, QueryIn Q, LayerOut O, const uint32_t* __restrict__ picks,
                                                      int64_t cap_q) {
  __shared__ uint8_t s_owner[8][32 * KMAX];
  __shared__ int32_t s_pre[8][32];
  __shared__ uint64_t s_key[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n = query_count(Q);
  const int64_t q0 = ((int64_t)blockIdx.x * 8 + w) * 32;
  if (q0 >= n) return;
  const int64_t q = q0 + lane;
  const int64_t base = O.offsets[q0];
  const int k = q < n ? (int)(O.offsets[q + 1] - O.offsets[q]) : 0;
  int incl = k;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int pre = incl - k, total = __shfl_sync(0xffffffffu, incl, 31);
  s_pre[w][lane] = pre;
  s_key[w][lane] = q < n ? (Q.keys ? Q.keys[q] : Q.key_base + (uint64_t)q) : 0;
  for (int i = 0; i < k; i++) s_owner[w][pre + i] = (uint8_t)lane;
  __syncwarp();
  constexpr int GU = GF_GATHER_UNROLL;
  int e = lane;
  for (; e + 32 * (GU - 1) < total; e += 32 * GU) {
    Slot sv[GU];
    int jv[GU];
#pragma unroll
    for (int u = 0; u < GU; u++) {
      jv[u] = s_owner[w][e + 32 * u];
      sv[u] = load_slot(GV.slots + picks[(e + 32 * u - s_pre[w][jv[u]]) * cap_q + q0 + jv[u]]);
    }
#pragma unroll
    for (int u = 0; u < GU; u++) store_out(O, base + e + 32 * u, sv[u], s_key[w][jv[u]], e + 32 * u - s_pre[w][jv[u]]);
  }
  for (; e < total; e += 32) {
    const int j = s_owner[w][e];
    const int i = e - s_pre[w][j];
    store_out(O, base + e, load_slot(GV.slots + picks[i * cap_q + q0 + j]), s_key[w][j], i);
  }
}

// ============================== host side ====================================

// the layer totals into pinned host memory (mapped under unified addressing)
__global__ void k_totals_to_host(const int64_t* __restrict__ totals, int n, int64_t* host) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) host[i] = totals[i];
  __threadfence_system();
}

__global__ void k_total(const int64_t* offsets, const int64_t* n_dev, int64_t n, int64_t* total) {
  *total = offsets[n_dev ? *n_dev : n];
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

gf_status check_args(int64_t n, int64_t fanout, int policy, int64_t delta) {
  if (n < 0) return fail(GF_EINVAL, "negative query count");
  if (fanout < 1) return fail(GF_EINVAL, "fanout must be >= 1");                 // sampling.py:240-241
  if (policy < 0 || policy > 2) return fail(GF_EINVAL, "unknown policy kind");   // sampling.py:38-39
  if (policy == GF_POLICY_TIME_WINDOW && delta <= 0) return fail(GF_EINVAL, "time_window policy requires delta > 0");
  return GF_OK;
}

int64_t grid_for_queries(int64_t cap_q, int per_query_threads) {
  int64_t blocks = (cap_q * per_query_threads + THREADS - 1) / THREADS;
  return std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)num_sms() * 16));
}

// One layer: count -> scan -> total -> write.  cap_q bounds the query count
// (exact when Q.n_dev is NULL).  total: device slot for this layer's total.
bool fused_enabled() {
  static const bool on = getenv("GF_NO_FUSED") == nullptr;
  return on;
}

// total must already be zero (callers clear their totals once per call): a layer with no
// queries launches nothing that would write it.
// after deletions the fused path is k_sample_fused_del; its Floyd-first selection exists only there,
// so GF_NO_FUSED (the unfused A/B kernels) applies to graphs without deletions
bool uses_fused(const gf_graph* g, int64_t fanout) {
  return fanout <= KMAX && g->slot_cap < (1ll << 32) && (fused_enabled() || g->any_deleted);
}

int tile_threads(const gf_graph* g, int policy) {
  if (g->any_deleted) return GF_DEL_THREADS;
  return policy == GF_POLICY_RECENT ? fused_threads<true>() : fused_threads<false>();
}
int64_t tile_words(const gf_graph* g, int64_t cap_q, int policy) {  // status words + ticket
  return (cap_q + tile_threads(g, policy) - 1) / tile_threads(g, policy) + 1;
}

// tile_state: (tiles + 1) zeroed words for the fused kernel, or NULL to allocate them here
gf_status layer_launch(gf_graph* g, const QueryIn& Q, int64_t cap_q, int64_t* d_offsets, const LayerOut& O, int64_t* total,
                       cudaStream_t s, uint64_t* tile_state = nullptr) {
  GraphView GV = view_of(g);
  const bool fast = !g->any_deleted;
  if (uses_fused(g, Q.fanout) && cap_q > 0) {
    // offsets[0] is written by tile 0, which always runs
    const int ft = tile_threads(g, Q.policy);
    const int64_t tiles = (cap_q + ft - 1) / ft;
    Scratch sb(s);
    if (!tile_state) {
      GF_TRY(sb.alloc(sizeof(uint64_t) * (tiles + 1)));
      tile_state = sb.as<uint64_t>();
      GF_CUDA(cudaMemsetAsync(tile_state, 0, sizeof(uint64_t) * (tiles + 1), s));
    }
    TileCtl C{tile_state, reinterpret_cast<unsigned long long*>(tile_state + tiles), total};
    if (g->any_deleted && Q.policy != GF_POLICY_RECENT) {  // split: select, scan, gather
      Scratch ps(s);
      GF_TRY(ps.alloc(sizeof(int64_t) * (size_t)cap_q + sizeof(uint32_t) * KMAX * (size_t)cap_q + 256));
      int64_t* counts = ps.as<int64_t>();
      uint32_t* picks = reinterpret_cast<uint32_t*>(counts + cap_q);
      GF_LAUNCH(k_sample_fused_del<true>, tiles, ft, 0, s, GV, Q, O, C, counts, picks, cap_q);
      GF_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), s));
      GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, counts, d_offsets + 1, cap_q, s); }, s));
      GF_LAUNCH(k_total, 1, 1, 0, s, d_offsets, Q.n_dev, Q.n, total);
      GF_LAUNCH(k_gather_picks, (cap_q + 255) / 256, 256, 0, s, GV, Q, O, picks, cap_q);
      return GF_OK;
    }
    if (g->any_deleted) GF_LAUNCH(k_sample_fused_del<false>, tiles, ft, 0, s, GV, Q, O, C, nullptr, nullptr, cap_q);
    else if (Q.policy == GF_POLICY_RECENT) GF_LAUNCH(k_sample_fused<true>, tiles, ft, 0, s, GV, Q, O, C);
    else GF_LAUNCH(k_sample_fused<false>, tiles, ft, 0, s, GV, Q, O, C);
    return GF_OK;
  }
  GF_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), s));
  if (cap_q == 0) {
    GF_CUDA(cudaMemsetAsync(total, 0, sizeof(int64_t), s));
    return GF_OK;
  }
  Scratch sb(s);
  Arena A;
  const bool rej = !fast && Q.policy != GF_POLICY_RECENT && Q.fanout <= KREJ;
  GF_TRY(sb.alloc((size_t)cap_q * 8 * (8 + (rej ? Q.fanout : 0)) + 8192));
  A.base = sb.as<char>();
  QState S{A.take<int64_t>(cap_q), A.take<int64_t>(cap_q), A.take<int64_t>(cap_q), A.take<int64_t>(cap_q),
           A.take<int64_t>(cap_q), A.take<int64_t>(cap_q), A.take<int64_t>(cap_q),
           rej ? A.take<int64_t>(cap_q * Q.fanout) : nullptr};
  int64_t* counts = A.take<int64_t>(cap_q);
  if (fast) GF_LAUNCH(k_count_lane, grid_for_queries(cap_q, 1), THREADS, 0, s, GV, Q, S, counts, cap_q);
  else GF_LAUNCH(k_count_general, grid_for_queries(cap_q, 32), THREADS, 0, s, GV, Q, S, counts, cap_q);
  cudaEvent_t e0 = g_profile.load(std::memory_order_relaxed) ? prof_start(s) : nullptr;
  GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, counts, d_offsets + 1, cap_q, s); }, s));
  if (e0) prof_stop("cub_scan_offsets", s, e0);
  GF_LAUNCH(k_total, 1, 1, 0, s, d_offsets, Q.n_dev, Q.n, total);
  if (fast && Q.fanout <= KMAX && g->slot_cap < (1ll << 32))
    GF_LAUNCH(k_write_coop, grid_for_queries(cap_q, 1), THREADS, 0, s, GV, Q, S, O);
  else if (fast)
    GF_LAUNCH(k_write_fast, grid_for_queries(cap_q, WG), THREADS, 0, s, GV, Q, S, O);
  if (!fast) GF_LAUNCH(k_write_general, grid_for_queries(cap_q, 32), THREADS, 0, s, GV, Q, S, O);
  return GF_OK;
}

}  // namespace

extern "C" {

#if GF_DEL_STATS
__attribute__((visibility("default"))) int gf_ab_del_stats(unsigned long long* host) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(host, g_del_stats, sizeof(unsigned long long) * 8);
}
#endif
#if GF_AB_TRACE
// measurement-only export of the A/B trace variant (not in include/gfb200.h)
__attribute__((visibility("default"))) int gf_ab_trace_dump(unsigned long long* host, int tiles) {
  if (tiles > TRACE_TILES) tiles = TRACE_TILES;
  return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * 5 * (size_t)tiles);
}
__attribute__((visibility("default"))) int gf_ab_trace_clear() {
  static unsigned long long z[TRACE_TILES][5];
  return (int)cudaMemcpyToSymbol(g_trace, z, sizeof(z));
}
#endif

gf_status gf_sample_layer(gf_graph* g, const int64_t* d_src, const int64_t* d_t_start, const int64_t* d_t_end, int64_t n,
                          int64_t fanout, int policy, int64_t delta, uint64_t seed, const uint64_t* d_keys,
                          uint64_t key_base, int64_t* d_offsets, int64_t* d_nbr, int64_t* d_eid, int64_t* d_ts,
                          uint64_t* d_out_keys, int64_t out_cap, int64_t* h_out_total, void* stream) {
  if (!g || !h_out_total || !d_offsets) return fail(GF_EINVAL, "NULL argument");
  GF_TRY(check_args(n, fanout, policy, delta));
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  *h_out_total = 0;
  Scratch sb(s);
  GF_TRY(sb.alloc(64));
  int64_t* total = sb.as<int64_t>();
  int* overflow = reinterpret_cast<int*>(total + 1);
  GF_CUDA(cudaMemsetAsync(total, 0, 16, s));
  QueryIn Q{d_src, d_t_start, d_t_end, d_keys, key_base, n, nullptr, fanout, policy, delta, seed};
  LayerOut O{d_offsets, d_nbr, d_eid, d_ts, d_out_keys, out_cap, overflow, 0};
  GF_TRY(layer_launch(g, Q, n, d_offsets, O, total, s));
  int64_t h[2] = {0, 0};
  GF_CUDA(cudaMemcpyAsync(h, total, 16, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  *h_out_total = h[0];
  if ((int)h[1] || h[0] > out_cap) return fail(GF_ERANGE, "output buffer too small");
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
  int64_t key_cap = 0;
  if (need_keys)
    for (int h = 0; h + 1 < n_hops; h++) key_cap = std::max(key_cap, h_caps[h]);
  // one region: totals, then every hop's tile state (zeroed by one memset), then the child keys
  int64_t zero_words = n_hops + 2;
  std::vector<int64_t> tile_off(n_hops, -1);
  for (int h = 0; h < n_hops; h++) {
    const int64_t cq = (h == 0) ? n_roots : h_caps[h - 1];
    if (uses_fused(g, h_fanouts[h]) && cq > 0) {
      tile_off[h] = zero_words;
      zero_words += tile_words(g, cq, policy);
    }
  }
  const size_t bytes = sizeof(int64_t) * (size_t)zero_words + 256 + 2 * sizeof(uint64_t) * (size_t)key_cap + 512;
  Scratch sb(s);
  char* base = nullptr;
  int64_t* hbuf = nullptr;
  std::vector<int64_t> hvec;
  const bool own = g->smp_busy.exchange(1) == 0;  // the persistent buffer, unless another call holds it
  struct Release {
    gf_graph* g;
    bool own;
    ~Release() {
      if (own) g->smp_busy.store(0);
    }
  } rel{g, own};
  if (own) {
    if (bytes > g->smp_bytes) {
      if (g->smp_buf) GF_CUDA(cudaFreeAsync(g->smp_buf, s));
      g->smp_buf = nullptr;
      g->smp_bytes = 0;
      GF_CUDA(cudaMallocAsync(&g->smp_buf, bytes + bytes / 4, s));
      g->smp_bytes = bytes + bytes / 4;
    }
    if (!g->smp_host) GF_CUDA(cudaMallocHost(&g->smp_host, 4096));
    base = (char*)g->smp_buf;
    if (n_hops + 1 <= 512) hbuf = g->smp_host;
  } else {
    GF_TRY(sb.alloc(bytes));
    base = sb.as<char>();
  }
  if (!hbuf) {
    hvec.resize(n_hops + 1);
    hbuf = hvec.data();
  }
  int64_t* totals = reinterpret_cast<int64_t*>(base);
  uint64_t* keys0 = reinterpret_cast<uint64_t*>(base + ((sizeof(int64_t) * zero_words + 255) & ~size_t(255)));
  uint64_t* keybuf[2] = {keys0, keys0 + key_cap};
  int* overflow = reinterpret_cast<int*>(totals + n_hops);
  GF_CUDA(cudaMemsetAsync(totals, 0, sizeof(int64_t) * zero_words, s));
  const int64_t* src = d_roots;
  const int64_t* tend = d_ts;
  const int64_t* n_dev = nullptr;
  const uint64_t* in_keys = nullptr;
  for (int h = 0; h < n_hops; h++) {
    uint64_t* out_keys = (need_keys && h + 1 < n_hops) ? keybuf[h & 1] : nullptr;
    int64_t cap_q = (h == 0) ? n_roots : h_caps[h - 1];
    QueryIn Q{src, nullptr, tend, in_keys, root_key_base, n_roots, n_dev, h_fanouts[h], policy, delta,
              gf::seed_sequence_2(seed, h)};
    LayerOut O{d_offsets[h], d_nbr[h], d_eid[h], d_ts_out[h], out_keys, h_caps[h], overflow, h == n_hops - 1};
    if (g_profile.load(std::memory_order_relaxed))
      g_prof_tag = std::string(policy == GF_POLICY_RECENT ? "recent" : policy == GF_POLICY_UNIFORM ? "uniform" : "tw") +
                   "/hop" + std::to_string(h);
    gf_status st = layer_launch(g, Q, cap_q, d_offsets[h], O, totals + h, s,
                                tile_off[h] >= 0 ? reinterpret_cast<uint64_t*>(totals + tile_off[h]) : nullptr);
    g_prof_tag.clear();
    GF_TRY(st);
    src = d_nbr[h];
    tend = d_ts_out[h];
    n_dev = totals + h;
    in_keys = out_keys;
  }
  int64_t* h = hbuf;
  if (h == g->smp_host) {
    // the pinned totals are written by a kernel (zero-copy): a DMA copy would queue behind the
    // caller's own D2H of earlier results on the copy engine and stall this return
    GF_LAUNCH(k_totals_to_host, 1, 32, 0, s, totals, n_hops + 1, h);
  } else {
    GF_CUDA(cudaMemcpyAsync(h, totals, sizeof(int64_t) * (n_hops + 1), cudaMemcpyDeviceToHost, s));
  }
  GF_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < n_hops; i++) h_totals[i] = h[i];
  if ((int)h[n_hops]) return fail(GF_ERANGE, "output buffer too small");
  for (int i = 0; i < n_hops; i++)
    if (h[i] > h_caps[i]) return fail(GF_ERANGE, "output buffer too small");
  return GF_OK;
}

}  // extern "C"
