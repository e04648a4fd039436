// gf_cache.cu -- vectorised dynamic feature cache (K4/K5), row gather (K6),
// feature tables (K7) and the harness fetch block.
//
// Replaces VectorCache (reference cache.py:55-233), NodeFeatureTable.get /
// EdgeFeatureTable.get (features.py:49-58, 107-120) and the per-minibatch
// fetch block of the harness (harness.py:438-446).  Cache state (keys,
// scores, rows, fifo_head, hit/miss/eviction counters) is device-resident and
// evolves exactly as the reference's (bit-exact scores, slots and rows).
//
// key -> slot map: open addressing (linear probing, splitmix64 hash) over a
// power-of-two table >= 2x capacity, rebuilt from keys[] after every insert.
// Rows are stored with a 16-byte aligned pitch so K6 moves them with 128-bit loads, staged in
// shared memory for packed outputs of any width.  The fetch block copies each output row once
// (hits from the cache, misses from the table) and synchronises with the host once.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "gf_common.cuh"

using namespace gf;

struct gf_cache {
  int device = 0;
  int policy = 0;
  int64_t capacity = 0, dim = 0, pitch = 0;
  double lam = 0.2;
  int64_t max_update = 0;
  int64_t fifo_head = 0;
  int64_t *keys = nullptr, *scores = nullptr;
  float* storage = nullptr;
  int64_t tsize = 0;
  int64_t* hkeys = nullptr;
  int32_t* hslots = nullptr;
  long long* counters = nullptr;  // hits, misses, evictions
  long long* hsmall = nullptr;    // pinned: the fetch block's counts read back
};

struct gf_cache_snap {
  int policy;
  int64_t capacity, dim, pitch, fifo_head;
  int64_t *keys, *scores;
  float* storage;
};

struct gf_ftable {
  int device = 0;
  int kind = 0;  // 0 node (dense by id), 1 edge (sorted ids)
  int64_t dim = 0, pitch = 0;
  int64_t n = 0, cap = 0;        // node: id capacity; edge: rows
  float* rows = nullptr;
  uint8_t* present = nullptr;    // node
  int64_t* ids = nullptr;        // edge (sorted)
  int64_t last_id = INT64_MIN;   // edge
  int64_t count = 0;             // node: number of present ids
};

namespace {

__device__ __forceinline__ uint64_t hash_key(int64_t k) { return splitmix64((uint64_t)k); }

__device__ __forceinline__ int32_t map_find(const int64_t* __restrict__ hk, const int32_t* __restrict__ hs, int64_t tmask,
                                            int64_t key) {
  uint64_t h = hash_key(key) & tmask;
  while (true) {
    int64_t k = hk[h];
    if (k == key) return hs[h];
    if (k == GF_EMPTY_KEY) return -1;
    h = (h + 1) & tmask;
  }
}

__global__ void k_map_clear(int64_t* hk, int64_t t) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < t; i += (int64_t)gridDim.x * blockDim.x)
    hk[i] = GF_EMPTY_KEY;
}

__global__ void k_map_build(const int64_t* __restrict__ keys, int64_t cap, int64_t* hk, int32_t* hs, int64_t tmask) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cap; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t key = keys[s];
    if (key == GF_EMPTY_KEY) continue;
    uint64_t h = hash_key(key) & tmask;
    while (true) {
      unsigned long long prev = atomicCAS((unsigned long long*)&hk[h], (unsigned long long)GF_EMPTY_KEY,
                                          (unsigned long long)key);
      if (prev == (unsigned long long)GF_EMPTY_KEY) {
        hs[h] = (int32_t)s;
        break;
      }
      h = (h + 1) & tmask;
    }
  }
}

// K4: probe every key; hit mask + slot, and hit count
__global__ void k_lookup(const int64_t* __restrict__ keys, int64_t n, const int64_t* __restrict__ hk,
                         const int32_t* __restrict__ hs, int64_t tmask, int32_t* slots, uint8_t* hit, long long* hits) {
  long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = map_find(hk, hs, tmask, keys[i]);
    slots[i] = s;
    if (hit) hit[i] = s >= 0;
    c += s >= 0;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)hits, (unsigned long long)c);
}

// LRU batch scoring: every occupied score -1 once per call (cache.py:106-107)
__global__ void k_lru_decay(const int64_t* __restrict__ keys, int64_t* scores, int64_t cap) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cap; s += (int64_t)gridDim.x * blockDim.x)
    if (keys[s] != GF_EMPTY_KEY) scores[s] -= 1;
}
// then hit slots = 0 (cache.py:108) / LFU += multiplicity (cache.py:109-111)
__global__ void k_score_hits(const int32_t* __restrict__ slots, int64_t n, int64_t* scores, int lfu) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = slots[i];
    if (s < 0) continue;
    if (lfu) atomicAdd((unsigned long long*)&scores[s], 1ull);
    else scores[s] = 0;
  }
}

// first-occurrence dedupe of the masked keys (stable): a scratch hash set holding
// the smallest index per key
__global__ void k_first_insert(const int64_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ slots,
                               int64_t* sk, long long* smin, int64_t smask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (slots && slots[i] >= 0) continue;
    int64_t key = keys[i];
    uint64_t h = hash_key(key) & smask;
    while (true) {
      unsigned long long prev = atomicCAS((unsigned long long*)&sk[h], (unsigned long long)GF_EMPTY_KEY,
                                          (unsigned long long)key);
      if (prev == (unsigned long long)GF_EMPTY_KEY || (int64_t)prev == key) {
        atomicMin(&smin[h], (long long)i);
        break;
      }
      h = (h + 1) & smask;
    }
  }
}

__device__ __forceinline__ int64_t set_find(const int64_t* sk, int64_t smask, int64_t key) {
  uint64_t h = hash_key(key) & smask;
  while (sk[h] != key) h = (h + 1) & smask;
  return (int64_t)h;
}

__global__ void k_first_flags(const int64_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ slots,
                              const int64_t* __restrict__ sk, const long long* __restrict__ smin, int64_t smask, int64_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t f = 0;
    if (!(slots && slots[i] >= 0)) f = (smin[set_find(sk, smask, keys[i])] == i);
    flag[i] = f;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) flag[n] = 0;
}

// scatter first occurrences to their rank; also map every miss occurrence to its rank
__global__ void k_first_scatter(const int64_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ slots,
                                const int64_t* __restrict__ flag, const int64_t* __restrict__ pos, const int64_t* __restrict__ sk,
                                const long long* __restrict__ smin, int64_t smask, int64_t* out_keys, int64_t* out_src,
                                int64_t* miss_rank) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (flag[i]) {
      out_keys[pos[i]] = keys[i];
      if (out_src) out_src[pos[i]] = i;
    }
    if (miss_rank) {
      if (slots && slots[i] >= 0) miss_rank[i] = -1;
      else miss_rank[i] = pos[smin[set_find(sk, smask, keys[i])]];
    }
  }
}

// K6: row gather out[i] = table[idx[i]] (zeros for idx < 0); warp per row
__global__ void k_gather_rows(const float* __restrict__ table, int64_t ld, const int64_t* __restrict__ idx32_or_64,
                              const int32_t* __restrict__ idx32, int64_t n, int64_t dim, float* __restrict__ out,
                              int64_t out_ld) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = ((ld & 3) == 0) && ((out_ld & 3) == 0) && ((dim & 3) == 0) &&
                   ((((uintptr_t)table) & 15) == 0) && ((((uintptr_t)out) & 15) == 0);
  for (int64_t i = warp; i < n; i += nw) {
    int64_t r = idx32 ? (int64_t)idx32[i] : idx32_or_64[i];
    float* o = out + i * out_ld;
    if (vec) {
      float4* o4 = reinterpret_cast<float4*>(o);
      if (r < 0) {
        for (int64_t c = lane; c < dim / 4; c += 32) o4[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        const float4* t4 = reinterpret_cast<const float4*>(table + r * ld);
        for (int64_t c = lane; c < dim / 4; c += 32) o4[c] = __ldg(t4 + c);
      }
    } else {
      if (r < 0) {
        for (int64_t c = lane; c < dim; c += 32) o[c] = 0.f;
      } else {
        const float* t = table + r * ld;
        for (int64_t c = lane; c < dim; c += 32) o[c] = __ldg(t + c);
      }
    }
  }
}

int64_t pow2_at_least(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
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

// K6 (fetch block): out[i] = cache row (slot >= 0), else table row (tidx >= 0), else zeros.  One warp
// per row: every 128-bit load of the 16-byte-pitched source row is issued before any use, the row is
// staged in shared memory, then written to the packed [n, dim] output with coalesced stores (any
// dim alignment).
constexpr int FG_V4 = 8;  // float4 per lane: rows up to 1024 floats
__global__ void __launch_bounds__(256) k_fetch_gather(const float* __restrict__ cache, int64_t cpitch,
                                                      const int32_t* __restrict__ slots, const float* __restrict__ table,
                                                      int64_t tpitch, const int64_t* __restrict__ tidx, int64_t n,
                                                      int64_t dim, float* __restrict__ out) {
  __shared__ float4 sm[8][32 * FG_V4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int dim4 = (int)((dim + 3) >> 2);
  const float* smf = reinterpret_cast<const float*>(sm[w]);
  for (int64_t i = warp; i < n; i += nw) {
    const int32_t sl = slots ? slots[i] : -1;
    const float4* src = nullptr;
    if (sl >= 0) src = reinterpret_cast<const float4*>(cache + (int64_t)sl * cpitch);
    else if (tidx && tidx[i] >= 0) src = reinterpret_cast<const float4*>(table + tidx[i] * tpitch);
    float4 v[FG_V4];
#pragma unroll
    for (int k = 0; k < FG_V4; k++) {
      const int c4 = lane + 32 * k;
      v[k] = (src && c4 < dim4) ? __ldg(src + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < FG_V4; k++)
      if (lane + 32 * k < dim4) sm[w][lane + 32 * k] = v[k];
    __syncwarp();
    float* o = out + i * dim;
    for (int64_t c = lane; c < dim; c += 32) __stcs(o + c, smf[c]);
    __syncwarp();
  }
}

gf_status gather(const float* table, int64_t ld, const int64_t* idx64, const int32_t* idx32, int64_t n, int64_t dim,
                 float* out, int64_t out_ld, cudaStream_t s) {
  if (n <= 0 || dim <= 0) return GF_OK;
  if (out_ld == dim && (ld & 3) == 0 && (((uintptr_t)table) & 15) == 0 && dim <= 4 * 32 * FG_V4) {
    // staged 128-bit path (rows of a 16-byte pitch, packed output of any alignment)
    const int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 16);
    GF_LAUNCH(k_fetch_gather, blocks, 256, 0, s, table, ld, idx32, table, ld, idx64, n, dim, out);
    return GF_OK;
  }
  int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 32);
  GF_LAUNCH(k_gather_rows, blocks, 256, 0, s, table, ld, idx64, idx32, n, dim, out, out_ld);
  return GF_OK;
}

gf_status rebuild_map(gf_cache* c, cudaStream_t s) {
  const int64_t G = 4 * num_sms();
  GF_LAUNCH(k_map_clear, grid_for(c->tsize, 256, G), 256, 0, s, c->hkeys, c->tsize);
  GF_LAUNCH(k_map_build, grid_for(c->capacity, 256, G), 256, 0, s, c->keys, c->capacity, c->hkeys, c->hslots, c->tsize - 1);
  return GF_OK;
}

// Stable first-occurrence dedupe of keys[i] where slots[i] < 0 (all keys if slots == NULL).
// Writes the unique keys (in first-occurrence order) to out_keys, their source
// indices to out_src (optional), per-occurrence rank to miss_rank (optional);
// returns the count in *h_count (synchronises).
gf_status dedupe_first(const int64_t* keys, int64_t n, const int32_t* slots, int64_t* out_keys, int64_t* out_src,
                       int64_t* miss_rank, int64_t* h_count, cudaStream_t s) {
  *h_count = 0;
  if (n == 0) return GF_OK;
  int64_t ssize = pow2_at_least(2 * n);
  Scratch sb(s);
  Arena A;
  GF_TRY(sb.alloc((size_t)ssize * 16 + (size_t)(n + 1) * 16 + 4096));
  A.base = sb.as<char>();
  int64_t* sk = A.take<int64_t>(ssize);
  long long* smin = A.take<long long>(ssize);
  int64_t* flag = A.take<int64_t>(n + 1);
  int64_t* pos = A.take<int64_t>(n + 1);
  const int64_t G = 8 * num_sms();
  GF_CUDA(cudaMemsetAsync(sk, 0xff, (size_t)ssize * 8, s));      // EMPTY_KEY = -1
  GF_CUDA(cudaMemsetAsync(smin, 0x7f, (size_t)ssize * 8, s));    // large
  GF_LAUNCH(k_first_insert, grid_for(n, 256, G), 256, 0, s, keys, n, slots, sk, smin, ssize - 1);
  GF_LAUNCH(k_first_flags, grid_for(n, 256, G), 256, 0, s, keys, n, slots, sk, smin, ssize - 1, flag);
  GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, flag, pos, (int)(n + 1), s); }, s));
  GF_LAUNCH(k_first_scatter, grid_for(n, 256, G), 256, 0, s, keys, n, slots, flag, pos, sk, smin, ssize - 1, out_keys,
            out_src, miss_rank);
  GF_CUDA(cudaMemcpyAsync(h_count, pos + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

__global__ void k_add_counter(long long* ctr, long long v) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *ctr += v;
}

__global__ void k_any_hit(const int32_t* slots, int64_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (slots[i] >= 0) *flag = 1;
}

// place admitted keys: target slot per admitted row, new score, row copy
__global__ void k_place(const int64_t* __restrict__ akeys, const int64_t* __restrict__ asrc, const int64_t* __restrict__ aslot,
                        int64_t na, int64_t* keys, int64_t* scores, int64_t score, long long* evictions, int count_evictions) {
  long long ev = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < na; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = aslot[j];
    if (count_evictions && keys[s] != GF_EMPTY_KEY) ev++;
    keys[s] = akeys[j];
    scores[s] = score;
  }
  for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
  if ((threadIdx.x & 31) == 0 && ev) atomicAdd((unsigned long long*)evictions, (unsigned long long)ev);
}

__global__ void k_copy_rows_to_slots(const float* __restrict__ values, int64_t dim, const int64_t* __restrict__ asrc,
                                     const int64_t* __restrict__ aslot, int64_t na, float* storage, int64_t pitch) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < na; j += nw) {
    const float* src = values + asrc[j] * dim;
    float* dst = storage + aslot[j] * pitch;
    for (int64_t c = lane; c < dim; c += 32) dst[c] = src[c];
  }
}

__global__ void k_fifo_slots(int64_t head, int64_t cap, int64_t na, int64_t* aslot) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < na; j += (int64_t)gridDim.x * blockDim.x)
    aslot[j] = (head + j) % cap;
}

// free-slot flags and the score range of the occupied slots
__global__ void k_free_flags(const int64_t* keys, const int64_t* scores, int64_t cap, int64_t* flag, long long* mm) {
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cap; s += (int64_t)gridDim.x * blockDim.x) {
    const bool empty = keys[s] == GF_EMPTY_KEY;
    flag[s] = empty;
    if (!empty) {
      lo = min(lo, (long long)scores[s]);
      hi = max(hi, (long long)scores[s]);
    }
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0 && lo <= hi) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) flag[cap] = 0;
}
__global__ void k_free_scatter(const int64_t* flag, const int64_t* pos, int64_t cap, int64_t* free_slots) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cap; s += (int64_t)gridDim.x * blockDim.x)
    if (flag[s]) free_slots[pos[s]] = s;
}
// score - lo: order-preserving and narrow, so the victim sort runs over only the bits the range needs;
// the sort's values (slot ids) are written in the same pass
__global__ void k_score_keys(const int64_t* scores, int64_t cap, int64_t lo, uint64_t* out, uint32_t* iota) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cap; s += (int64_t)gridDim.x * blockDim.x) {
    out[s] = (uint64_t)(scores[s] - lo);
    iota[s] = (uint32_t)s;
  }
}
__global__ void k_victims(const uint32_t* sorted_slots, int64_t r, int64_t* aslot) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < r; j += (int64_t)gridDim.x * blockDim.x)
    aslot[j] = sorted_slots[j];
}

// free-slot state computed ahead of the placement (fetch block: read back with its other counts)
struct FreeState {
  const int64_t* free_slots;  // ascending free slots
  int64_t nfree;
  long long lo, hi;           // score range of the occupied slots (LLONG_MAX/MIN when none)
};

gf_status place_impl(gf_cache* c, const int64_t* ukeys, const int64_t* usrc, int64_t u, const float* values,
                     int64_t* h_admitted, cudaStream_t s, const FreeState* pre = nullptr);

gf_status insert_impl(gf_cache* c, const int64_t* keys, int64_t n, const float* values, int64_t* h_admitted, cudaStream_t s) {
  *h_admitted = 0;
  if (n == 0) return GF_OK;
  const int64_t G = 8 * num_sms();
  Scratch sb(s);
  Arena A;
  GF_TRY(sb.alloc((size_t)n * 4 + (size_t)n * 8 * 2 + 64 + 4096));
  A.base = sb.as<char>();
  int32_t* slots = A.take<int32_t>(n);
  int64_t* ukeys = A.take<int64_t>(n);
  int64_t* usrc = A.take<int64_t>(n);
  int* flag = A.take<int>(1);
  long long* dummy = A.take<long long>(1);
  GF_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  GF_CUDA(cudaMemsetAsync(dummy, 0, sizeof(long long), s));
  GF_LAUNCH(k_lookup, grid_for(n, 256, G), 256, 0, s, keys, n, c->hkeys, c->hslots, c->tsize - 1, slots, (uint8_t*)nullptr, dummy);
  GF_LAUNCH(k_any_hit, grid_for(n, 256, G), 256, 0, s, slots, n, flag);
  int already = 0;
  GF_CUDA(cudaMemcpyAsync(&already, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  if (already) return fail(GF_EINVAL, "a key is already cached");  // cache.py:139-140
  int64_t u = 0;
  GF_TRY(dedupe_first(keys, n, nullptr, ukeys, usrc, nullptr, &u, s));
  return place_impl(c, ukeys, usrc, u, values, h_admitted, s);
}

// Admit the first min(u, max_update) of u distinct, uncached keys (cache.py:144-177); the row of
// ukeys[j] is values[usrc[j]].
gf_status place_impl(gf_cache* c, const int64_t* ukeys, const int64_t* usrc, int64_t u, const float* values,
                     int64_t* h_admitted, cudaStream_t s, const FreeState* pre) {
  *h_admitted = 0;
  const int64_t G = 8 * num_sms();
  int64_t na = std::min<int64_t>(u, c->max_update);  // cache.py:144
  if (na == 0) return GF_OK;
  Scratch ab(s);
  GF_TRY(ab.alloc((size_t)na * 8 + 256));
  int64_t* aslot = ab.as<int64_t>();
  const int64_t new_score = (c->policy == GF_CACHE_LFU) ? 1 : 0;
  if (c->policy == GF_CACHE_FIFO) {  // cache.py:148-153
    GF_LAUNCH(k_fifo_slots, grid_for(na, 256, G), 256, 0, s, c->fifo_head, c->capacity, na, aslot);
    GF_LAUNCH(k_place, grid_for(na, 256, G), 256, 0, s, ukeys, usrc, aslot, na, c->keys, c->scores, (int64_t)0,
              c->counters + 2, 1);
    c->fifo_head = (c->fifo_head + na) % c->capacity;
  } else {
    // free slots ascending (cache.py:155-159)
    const int64_t cap = c->capacity;
    Scratch fb(s);
    Arena F;
    GF_TRY(fb.alloc((size_t)(cap + 1) * 8 * 3 + (size_t)cap * 4 * 2 + (size_t)cap * 8 * 2 + 8192));
    F.base = fb.as<char>();
    int64_t* ff = F.take<int64_t>(cap + 1);
    int64_t* fpos = F.take<int64_t>(cap + 1);
    int64_t* free_slots = F.take<int64_t>(cap + 1);
    uint32_t* iota = F.take<uint32_t>(cap);
    uint32_t* sorted_slots = F.take<uint32_t>(cap);
    uint64_t* skeys = F.take<uint64_t>(cap);
    uint64_t* skeys_sorted = F.take<uint64_t>(cap);
    int64_t nfree = 0;
    long long hmm[2];
    if (pre) {
      free_slots = const_cast<int64_t*>(pre->free_slots);
      nfree = pre->nfree;
      hmm[0] = pre->lo;
      hmm[1] = pre->hi;
    } else {
      long long* mm = reinterpret_cast<long long*>(F.take<int64_t>(2));
      const long long mm0[2] = {LLONG_MAX, LLONG_MIN};
      GF_CUDA(cudaMemcpyAsync(mm, mm0, sizeof(mm0), cudaMemcpyHostToDevice, s));
      GF_LAUNCH(k_free_flags, grid_for(cap, 256, G), 256, 0, s, c->keys, c->scores, cap, ff, mm);
      GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, ff, fpos, (int)(cap + 1), s); }, s));
      GF_LAUNCH(k_free_scatter, grid_for(cap, 256, G), 256, 0, s, ff, fpos, cap, free_slots);
      GF_CUDA(cudaMemcpyAsync(&nfree, fpos + cap, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      GF_CUDA(cudaMemcpyAsync(hmm, mm, sizeof(hmm), cudaMemcpyDeviceToHost, s));
      GF_CUDA(cudaStreamSynchronize(s));
    }
    int64_t nfill = std::min(nfree, na);
    if (nfill > 0) {
      GF_LAUNCH(k_place, grid_for(nfill, 256, G), 256, 0, s, ukeys, usrc, free_slots, nfill, c->keys, c->scores, new_score,
                c->counters + 2, 0);
      GF_LAUNCH(k_copy_rows_to_slots, grid_for(nfill * 32, 256, G), 256, 0, s, values, c->dim, usrc, free_slots, nfill,
                c->storage, c->pitch);
    }
    int64_t r = na - nfill;
    if (r > 0) {
      // victims: lowest (score, slot) over the post-fill occupied slots (cache.py:160-166)
      // post-fill scores: the occupied range plus the new slots' score
      const long long lo = std::min<long long>(hmm[0], new_score), hi = std::max<long long>(hmm[1], new_score);
      int bits = 1;
      while (bits < 64 && ((unsigned long long)(hi - lo) >> bits) != 0) bits++;
      GF_LAUNCH(k_score_keys, grid_for(cap, 256, G), 256, 0, s, c->scores, cap, (int64_t)lo, skeys, iota);
      cudaEvent_t e0 = g_profile.load(std::memory_order_relaxed) ? prof_start(s) : nullptr;
      GF_TRY(cub_call([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, skeys, skeys_sorted, iota, sorted_slots, (int)cap, 0, bits, s);
      }, s));
      if (e0) prof_stop("cub_victim_sort", s, e0);
      GF_LAUNCH(k_victims, grid_for(r, 256, G), 256, 0, s, sorted_slots, r, aslot);
      GF_LAUNCH(k_place, grid_for(r, 256, G), 256, 0, s, ukeys + nfill, usrc + nfill, aslot, r, c->keys, c->scores,
                new_score, c->counters + 2, 1);
      GF_LAUNCH(k_copy_rows_to_slots, grid_for(r * 32, 256, G), 256, 0, s, values, c->dim, usrc + nfill, aslot, r,
                c->storage, c->pitch);
    }
    GF_TRY(rebuild_map(c, s));
    *h_admitted = na;
    if (!pre) GF_CUDA(cudaStreamSynchronize(s));  // the fetch block stays stream-ordered
    return GF_OK;
  }
  GF_LAUNCH(k_copy_rows_to_slots, grid_for(na * 32, 256, G), 256, 0, s, values, c->dim, usrc, aslot, na, c->storage, c->pitch);
  GF_TRY(rebuild_map(c, s));
  *h_admitted = na;
  if (!pre) GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status fetch_impl(gf_cache* c, const int64_t* keys, int64_t n, float* values, uint8_t* hit, int64_t* miss_keys,
                     int64_t* h_n_miss, int64_t* miss_rank, cudaStream_t s) {
  *h_n_miss = 0;
  if (n == 0) return GF_OK;  // cache.py:96-97: empty batch changes nothing
  const int64_t G = 8 * num_sms();
  Scratch sb(s);
  GF_TRY(sb.alloc((size_t)n * 4 + 256));
  int32_t* slots = sb.as<int32_t>();
  GF_LAUNCH(k_lookup, grid_for(n, 256, G), 256, 0, s, keys, n, c->hkeys, c->hslots, c->tsize - 1, slots, hit, c->counters);
  if (values) GF_TRY(gather(c->storage, c->pitch, nullptr, slots, n, c->dim, values, c->dim, s));
  if (c->policy == GF_CACHE_LRU) {
    GF_LAUNCH(k_lru_decay, grid_for(c->capacity, 256, G), 256, 0, s, c->keys, c->scores, c->capacity);
    GF_LAUNCH(k_score_hits, grid_for(n, 256, G), 256, 0, s, slots, n, c->scores, 0);
  } else if (c->policy == GF_CACHE_LFU) {
    GF_LAUNCH(k_score_hits, grid_for(n, 256, G), 256, 0, s, slots, n, c->scores, 1);
  }
  int64_t nm = 0;
  GF_TRY(dedupe_first(keys, n, slots, miss_keys, nullptr, miss_rank, &nm, s));
  *h_n_miss = nm;
  return GF_OK;
}

__global__ void k_count_misses(const uint8_t* hit, const int32_t* dummy, int64_t n, long long* misses) {
  long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) c += !hit[i];
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)misses, (unsigned long long)c);
}

// ---- feature tables --------------------------------------------------------------
__global__ void k_node_winner(const int64_t* ids, int64_t n, long long* win) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicMax(&win[ids[i]], (long long)i);
}
__global__ void k_node_put(const int64_t* ids, int64_t n, const long long* win, const float* rows, int64_t dim, float* table,
                           int64_t pitch, uint8_t* present, long long* newcount) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    int64_t id = ids[i];
    if (win[id] != i) continue;
    for (int64_t c = lane; c < dim; c += 32) table[id * pitch + c] = rows[i * dim + c];
    if (lane == 0) {
      if (!present[id]) atomicAdd((unsigned long long*)newcount, 1ull);
      present[id] = 1;
    }
  }
}
__global__ void k_node_idx(const int64_t* ids, int64_t n, int64_t cap, const uint8_t* present, int64_t* idx, uint8_t* found) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t id = ids[i];
    bool f = id >= 0 && id < cap && present[id];
    idx[i] = f ? id : -1;
    if (found) found[i] = f;
  }
}
// K7: sorted-id binary search (features.py:107-120)
__global__ void k_edge_idx(const int64_t* ids, int64_t n, const int64_t* __restrict__ sorted, int64_t m, int64_t* idx,
                           uint8_t* found) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t key = ids[i];
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (__ldg(sorted + mid) < key) lo = mid + 1;
      else hi = mid;
    }
    bool f = lo < m && __ldg(sorted + lo) == key;
    idx[i] = f ? lo : -1;
    if (found) found[i] = f;
  }
}
__global__ void k_edge_check(const int64_t* ids, int64_t n, int64_t last, int* bad, long long* mx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t prev = i ? ids[i - 1] : last;
    if ((i || last != INT64_MIN) && ids[i] <= prev) *bad = 1;
    if (i == n - 1) *mx = ids[i];
  }
}
__global__ void k_minmax_ids(const int64_t* ids, int64_t n, long long* mm) {
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    mn = min(mn, (long long)ids[i]);
    mx = max(mx, (long long)ids[i]);
  }
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], mn);
    atomicMax(&mm[1], mx);
  }
}
__global__ void k_copy_rows_packed(const float* src, int64_t n, int64_t dim, float* dst, int64_t pitch) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw)
    for (int64_t c = lane; c < dim; c += 32) dst[i * pitch + c] = src[i * dim + c];
}

template <class T>
gf_status grow(T*& p, int64_t keep, int64_t cap, cudaStream_t s, bool zero_tail = true, int64_t old_cap = 0) {
  T* q = nullptr;
  cudaError_t e = cudaMallocAsync(&q, sizeof(T) * (size_t)std::max<int64_t>(cap, 1), s);
  if (e != cudaSuccess) return fail(GF_ENOMEM, "device allocation failed");
  if (zero_tail) GF_CUDA(cudaMemsetAsync(q, 0, sizeof(T) * (size_t)std::max<int64_t>(cap, 1), s));
  if (p && keep > 0) GF_CUDA(cudaMemcpyAsync(q, p, sizeof(T) * (size_t)keep, cudaMemcpyDeviceToDevice, s));
  if (p) cudaFreeAsync(p, s);
  p = q;
  (void)old_cap;
  return GF_OK;
}


__global__ void k_fill_from_table(const int32_t* __restrict__ slots, const float* __restrict__ table, int64_t tpitch,
                                  const int64_t* __restrict__ tidx, int64_t n, int64_t dim, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    if (slots[i] >= 0 || tidx[i] < 0) continue;  // hit, or unknown id (zeros already written)
    const float* r = table + tidx[i] * tpitch;
    for (int64_t c = lane; c < dim; c += 32) out[i * dim + c] = __ldg(r + c);
  }
}



struct AddLL2 {
  __device__ __forceinline__ longlong2 operator()(const longlong2& a, const longlong2& b) const {
    return make_longlong2(a.x + b.x, a.y + b.y);
  }
};

// fetch block: per occurrence, {first occurrence of a missing key, ... and found in the table}
__global__ void k_ff_flags(const int64_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ slots,
                           const int64_t* __restrict__ sk, const long long* __restrict__ smin, int64_t smask,
                           const uint8_t* __restrict__ found, longlong2* flag2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    long long f = 0;
    if (slots[i] < 0) f = (smin[set_find(sk, smask, keys[i])] == i);
    flag2[i] = make_longlong2(f, f && found[i]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) flag2[n] = make_longlong2(0, 0);
}

// the found distinct misses in first-occurrence order, with the position of their first occurrence
__global__ void k_ff_scatter(const int64_t* __restrict__ keys, int64_t n, const longlong2* __restrict__ flag2,
                             const longlong2* __restrict__ pos2, int64_t* okeys, int64_t* osrc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag2[i].y) {
      okeys[pos2[i].y] = keys[i];
      osrc[pos2[i].y] = i;
    }
}

// {distinct misses, found distinct misses, free slots, occupied score min, max} for one readback
__global__ void k_ff_counts(const longlong2* pos2, int64_t n, const int64_t* fpos, int64_t cap, const long long* mm,
                            long long* out) {
  if (threadIdx.x || blockIdx.x) return;
  out[0] = pos2[n].x;
  out[1] = pos2[n].y;
  out[2] = fpos ? fpos[cap] : 0;
  out[3] = mm ? mm[0] : LLONG_MAX;
  out[4] = mm ? mm[1] : LLONG_MIN;
}

__global__ void k_mm_init(long long* mm) {
  if (threadIdx.x || blockIdx.x) return;
  mm[0] = LLONG_MAX;
  mm[1] = LLONG_MIN;
}

gf_status ftable_get_idx(gf_ftable* t, const int64_t* ids, int64_t n, int64_t* idx, uint8_t* found, cudaStream_t s) {
  const int64_t G = 8 * num_sms();
  if (t->kind == 0) {
    if (t->cap == 0) {
      GF_CUDA(cudaMemsetAsync(idx, 0xff, (size_t)n * 8, s));
      if (found) GF_CUDA(cudaMemsetAsync(found, 0, (size_t)n, s));
      return GF_OK;
    }
    GF_LAUNCH(k_node_idx, grid_for(n, 256, G), 256, 0, s, ids, n, t->cap, t->present, idx, found);
  } else {
    GF_LAUNCH(k_edge_idx, grid_for(n, 256, G), 256, 0, s, ids, n, t->ids, t->n, idx, found);
  }
  return GF_OK;
}

gf_status fetch_gather(gf_cache* c, const int32_t* slots, gf_ftable* t, const int64_t* tidx, int64_t n, float* out,
                       cudaStream_t s) {
  if (c->dim == 0) return GF_OK;
  if (c->dim > 4 * 32 * FG_V4) {  // wide rows: hits from the cache, then misses from the table
    GF_TRY(gather(c->storage, c->pitch, nullptr, slots, n, c->dim, out, c->dim, s));
    GF_LAUNCH(k_fill_from_table, grid_for(n * 32, 256, 8 * num_sms()), 256, 0, s, slots, t->rows, t->pitch, tidx, n,
              c->dim, out);
    return GF_OK;
  }
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 16);
  GF_LAUNCH(k_fetch_gather, blocks, 256, 0, s, c->storage, c->pitch, slots, t->rows, t->pitch, tidx, n, c->dim, out);
  return GF_OK;
}

}  // namespace

extern "C" {

gf_status gf_cache_create(int policy, int64_t capacity, int64_t dim, double lam, int device, gf_cache** out) {
  if (!out) return fail(GF_EINVAL, "out is NULL");
  *out = nullptr;
  if (policy < 0 || policy > 2) return fail(GF_EINVAL, "unknown cache policy");  // cache.py:57-58
  if (capacity < 1) return fail(GF_EINVAL, "capacity must be >= 1");           // cache.py:59-60
  if (!(lam > 0.0 && lam <= 1.0)) return fail(GF_EINVAL, "lam must be in (0, 1]");  // cache.py:61-62
  if (dim < 0) return fail(GF_EINVAL, "dim must be >= 0");
  if (capacity >= ((int64_t)1 << 31)) return fail(GF_EINVAL, "capacity must be < 2^31");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != device) cudaSetDevice(device);
  gf_cache* c = new gf_cache();
  c->device = device;
  c->policy = policy;
  c->capacity = capacity;
  c->dim = dim;
  c->pitch = (dim + 3) & ~int64_t(3);
  c->lam = lam;
  c->max_update = (int64_t)(lam * (double)capacity);  // cache.py:79-81: int(lam * capacity)
  c->tsize = pow2_at_least(std::max<int64_t>(2 * capacity, 64));
  cudaError_t e = cudaSuccess;
  e = (cudaError_t)(e | cudaMalloc(&c->keys, 8 * capacity));
  e = (cudaError_t)(e | cudaMalloc(&c->scores, 8 * capacity));
  e = (cudaError_t)(e | cudaMalloc(&c->storage, 4 * std::max<int64_t>(1, capacity * c->pitch)));
  e = (cudaError_t)(e | cudaMalloc(&c->hkeys, 8 * c->tsize));
  e = (cudaError_t)(e | cudaMalloc(&c->hslots, 4 * c->tsize));
  e = (cudaError_t)(e | cudaMalloc(&c->counters, 8 * 4));
  if (e != cudaSuccess) {
    gf_cache_destroy(c);
    if (cur != device) cudaSetDevice(cur);
    return fail(GF_ENOMEM, "cache allocation failed");
  }
  cudaMemset(c->keys, 0xff, 8 * capacity);
  cudaMemset(c->scores, 0, 8 * capacity);
  cudaMemset(c->storage, 0, 4 * std::max<int64_t>(1, capacity * c->pitch));
  cudaMemset(c->hkeys, 0xff, 8 * c->tsize);
  cudaMemset(c->counters, 0, 8 * 4);
  cudaDeviceSynchronize();
  if (cur != device) cudaSetDevice(cur);
  *out = c;
  return GF_OK;
}

gf_status gf_cache_destroy(gf_cache* c) {
  if (!c) return GF_OK;
  DeviceGuard dg(c->device);
  cudaFree(c->keys);
  cudaFree(c->scores);
  cudaFree(c->storage);
  cudaFree(c->hkeys);
  cudaFree(c->hslots);
  cudaFree(c->counters);
  if (c->hsmall) cudaFreeHost(c->hsmall);
  delete c;
  return GF_OK;
}

gf_status gf_cache_fetch(gf_cache* c, const int64_t* d_keys, int64_t n, float* d_values, uint8_t* d_hit, int64_t* d_miss_keys,
                         int64_t* h_n_miss, void* stream) {
  if (!c || !h_n_miss) return fail(GF_EINVAL, "NULL argument");
  if (n > 0 && (!d_keys || !d_hit || !d_miss_keys)) return fail(GF_EINVAL, "NULL array");
  DeviceGuard dg(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  GF_TRY(fetch_impl(c, d_keys, n, d_values, d_hit, d_miss_keys, h_n_miss, nullptr, s));
  if (n > 0)
    GF_LAUNCH(k_count_misses, grid_for(n, 256, 8 * num_sms()), 256, 0, s, d_hit, (const int32_t*)nullptr, n, c->counters + 1);
  return GF_OK;
}

gf_status gf_cache_insert(gf_cache* c, const int64_t* d_keys, int64_t n, const float* d_values, int64_t* h_admitted,
                          void* stream) {
  if (!c || !h_admitted) return fail(GF_EINVAL, "NULL argument");
  if (n > 0 && (!d_keys || !d_values)) return fail(GF_EINVAL, "NULL array");
  DeviceGuard dg(c->device);
  return insert_impl(c, d_keys, n, d_values, h_admitted, (cudaStream_t)stream);
}

gf_status gf_cache_stats(gf_cache* c, int64_t* h_hits, int64_t* h_misses, int64_t* h_evictions) {
  if (!c) return fail(GF_EINVAL, "NULL argument");
  DeviceGuard dg(c->device);
  // the fetch block's insert is stream-ordered and may still be counting evictions on any stream
  GF_CUDA(cudaDeviceSynchronize());
  long long v[4];
  GF_CUDA(cudaMemcpy(v, c->counters, sizeof(v), cudaMemcpyDeviceToHost));
  if (h_hits) *h_hits = v[0];
  if (h_misses) *h_misses = v[1];
  if (h_evictions) *h_evictions = v[2];
  return GF_OK;
}

gf_status gf_cache_reset_stats(gf_cache* c) {
  if (!c) return fail(GF_EINVAL, "NULL argument");
  DeviceGuard dg(c->device);
  GF_CUDA(cudaDeviceSynchronize());
  GF_CUDA(cudaMemset(c->counters, 0, 8 * 4));
  GF_CUDA(cudaDeviceSynchronize());
  return GF_OK;
}

gf_status gf_cache_get_state(gf_cache* c, int64_t* h_keys, int64_t* h_scores, float* h_storage, int64_t* h_fifo_head,
                             void* stream) {
  if (!c) return fail(GF_EINVAL, "NULL argument");
  DeviceGuard dg(c->device);
  // gf_fetch_features returns with its insert still queued on the caller's stream: order
  // against every stream, as gf_cache_stats does
  GF_CUDA(cudaDeviceSynchronize());
  cudaStream_t s = (cudaStream_t)stream;
  if (h_keys) GF_CUDA(cudaMemcpyAsync(h_keys, c->keys, 8 * c->capacity, cudaMemcpyDeviceToHost, s));
  if (h_scores) GF_CUDA(cudaMemcpyAsync(h_scores, c->scores, 8 * c->capacity, cudaMemcpyDeviceToHost, s));
  if (h_storage && c->dim > 0)
    GF_CUDA(cudaMemcpy2DAsync(h_storage, 4 * c->dim, c->storage, 4 * c->pitch, 4 * c->dim, c->capacity,
                              cudaMemcpyDeviceToHost, s));
  if (h_fifo_head) *h_fifo_head = c->fifo_head;
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_cache_set_state(gf_cache* c, const int64_t* h_keys, const int64_t* h_scores, const float* h_storage,
                             int64_t fifo_head, void* stream) {
  if (!c) return fail(GF_EINVAL, "NULL argument");
  if (fifo_head < 0 || fifo_head >= c->capacity) return fail(GF_EINVAL, "bad fifo head");  // before any copy
  DeviceGuard dg(c->device);
  GF_CUDA(cudaDeviceSynchronize());
  cudaStream_t s = (cudaStream_t)stream;
  if (h_keys) GF_CUDA(cudaMemcpyAsync(c->keys, h_keys, 8 * c->capacity, cudaMemcpyHostToDevice, s));
  if (h_scores) GF_CUDA(cudaMemcpyAsync(c->scores, h_scores, 8 * c->capacity, cudaMemcpyHostToDevice, s));
  if (h_storage && c->dim > 0)
    GF_CUDA(cudaMemcpy2DAsync(c->storage, 4 * c->pitch, h_storage, 4 * c->dim, 4 * c->dim, c->capacity,
                              cudaMemcpyHostToDevice, s));
  c->fifo_head = fifo_head;
  GF_TRY(rebuild_map(c, s));
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_cache_snapshot(gf_cache* c, gf_cache_snap** out, void* stream) {
  if (!c || !out) return fail(GF_EINVAL, "NULL argument");
  DeviceGuard dg(c->device);
  GF_CUDA(cudaDeviceSynchronize());
  cudaStream_t s = (cudaStream_t)stream;
  gf_cache_snap* p = new gf_cache_snap();
  p->policy = c->policy;
  p->capacity = c->capacity;
  p->dim = c->dim;
  p->pitch = c->pitch;
  p->fifo_head = c->fifo_head;
  size_t rows = 4 * (size_t)std::max<int64_t>(1, c->capacity * c->pitch);
  if (cudaMalloc(&p->keys, 8 * c->capacity) != cudaSuccess || cudaMalloc(&p->scores, 8 * c->capacity) != cudaSuccess ||
      cudaMalloc(&p->storage, rows) != cudaSuccess) {
    gf_cache_snapshot_free(p);
    return fail(GF_ENOMEM, "snapshot allocation failed");
  }
  GF_CUDA(cudaMemcpyAsync(p->keys, c->keys, 8 * c->capacity, cudaMemcpyDeviceToDevice, s));
  GF_CUDA(cudaMemcpyAsync(p->scores, c->scores, 8 * c->capacity, cudaMemcpyDeviceToDevice, s));
  GF_CUDA(cudaMemcpyAsync(p->storage, c->storage, rows, cudaMemcpyDeviceToDevice, s));
  GF_CUDA(cudaStreamSynchronize(s));
  *out = p;
  return GF_OK;
}

gf_status gf_cache_restore(gf_cache* c, const gf_cache_snap* p, void* stream) {
  if (!c || !p) return fail(GF_EINVAL, "NULL argument");
  if (p->policy != c->policy || p->capacity != c->capacity || p->dim != c->dim)  // cache.py:194-198
    return fail(GF_EINVAL, "snapshot shape does not match the cache");
  DeviceGuard dg(c->device);
  GF_CUDA(cudaDeviceSynchronize());
  cudaStream_t s = (cudaStream_t)stream;
  size_t rows = 4 * (size_t)std::max<int64_t>(1, c->capacity * c->pitch);
  GF_CUDA(cudaMemcpyAsync(c->keys, p->keys, 8 * c->capacity, cudaMemcpyDeviceToDevice, s));
  GF_CUDA(cudaMemcpyAsync(c->scores, p->scores, 8 * c->capacity, cudaMemcpyDeviceToDevice, s));
  GF_CUDA(cudaMemcpyAsync(c->storage, p->storage, rows, cudaMemcpyDeviceToDevice, s));
  c->fifo_head = p->fifo_head;
  GF_TRY(rebuild_map(c, s));
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_cache_snapshot_free(gf_cache_snap* p) {
  if (!p) return GF_OK;
  cudaFree(p->keys);
  cudaFree(p->scores);
  cudaFree(p->storage);
  delete p;
  return GF_OK;
}

gf_status gf_ftable_create(int kind, int64_t dim, int device, gf_ftable** out) {
  if (!out) return fail(GF_EINVAL, "out is NULL");
  if (kind != 0 && kind != 1) return fail(GF_EINVAL, "unknown feature table kind");
  if (dim < 0) return fail(GF_EINVAL, "dim must be >= 0");
  gf_ftable* t = new gf_ftable();
  t->device = device;
  t->kind = kind;
  t->dim = dim;
  t->pitch = (dim + 3) & ~int64_t(3);
  *out = t;
  return GF_OK;
}

gf_status gf_ftable_destroy(gf_ftable* t) {
  if (!t) return GF_OK;
  DeviceGuard dg(t->device);
  cudaFree(t->rows);
  cudaFree(t->present);
  cudaFree(t->ids);
  delete t;
  return GF_OK;
}

gf_status gf_ftable_size(gf_ftable* t, int64_t* h_n) {
  if (!t || !h_n) return fail(GF_EINVAL, "NULL argument");
  *h_n = t->kind == 0 ? t->count : t->n;
  return GF_OK;
}

gf_status gf_ftable_ids(gf_ftable* t, int64_t* d_ids, int64_t cap, int64_t* h_n, void* stream) {
  if (!t || !h_n) return fail(GF_EINVAL, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = t->kind == 0 ? t->count : t->n;
  *h_n = n;
  if (n > cap) return fail(GF_ERANGE, "id buffer too small");
  if (n == 0) return GF_OK;
  if (!d_ids) return fail(GF_EINVAL, "NULL id buffer");
  DeviceGuard dg(t->device);
  if (t->kind == 1) {
    GF_CUDA(cudaMemcpyAsync(d_ids, t->ids, 8 * n, cudaMemcpyDeviceToDevice, s));
  } else {
    // ascending ids whose present flag is set (stable selection over 0..cap-1)
    Scratch sb(s);
    size_t tmp = 0;
    GF_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, cub::CountingInputIterator<int64_t>(0), t->present, d_ids,
                                       (int64_t*)nullptr, t->cap, s));
    GF_TRY(sb.alloc(tmp + 64));
    int64_t* nsel = sb.as<int64_t>();
    GF_CUDA(cub::DeviceSelect::Flagged((char*)sb.p + 64, tmp, cub::CountingInputIterator<int64_t>(0), t->present,
                                       d_ids, nsel, t->cap, s));
  }
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_ftable_put(gf_ftable* t, const int64_t* d_ids, int64_t n, const float* d_rows, void* stream) {
  if (!t) return fail(GF_EINVAL, "NULL argument");
  if (n == 0) return GF_OK;
  DeviceGuard dg(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t G = 8 * num_sms();
  Scratch sb(s);
  GF_TRY(sb.alloc(64));
  long long* mm = sb.as<long long>();
  if (t->kind == 0) {
    long long init[2] = {LLONG_MAX, LLONG_MIN};
    GF_CUDA(cudaMemcpyAsync(mm, init, 16, cudaMemcpyHostToDevice, s));
    GF_LAUNCH(k_minmax_ids, grid_for(n, 256, G), 256, 0, s, d_ids, n, mm);
    GF_CUDA(cudaMemcpyAsync(init, mm, 16, cudaMemcpyDeviceToHost, s));
    GF_CUDA(cudaStreamSynchronize(s));
    if (init[0] < 0) return fail(GF_EINVAL, "node feature ids must be non-negative");
    int64_t need = init[1] + 1;
    if (need > t->cap) {
      int64_t nc = std::max<int64_t>(need, t->cap * 2);
      GF_TRY(grow(t->rows, t->cap * t->pitch, nc * t->pitch, s));
      GF_TRY(grow(t->present, t->cap, nc, s));
      t->cap = nc;
    }
    Scratch wb(s);
    GF_TRY(wb.alloc((size_t)t->cap * 8 + 64));
    long long* win = wb.as<long long>();
    long long* cnt = win + t->cap;
    GF_CUDA(cudaMemsetAsync(win, 0xff, (size_t)t->cap * 8 + 8, s));
    GF_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
    GF_LAUNCH(k_node_winner, grid_for(n, 256, G), 256, 0, s, d_ids, n, win);
    GF_LAUNCH(k_node_put, grid_for(n * 32, 256, G), 256, 0, s, d_ids, n, win, d_rows, t->dim, t->rows, t->pitch, t->present,
              cnt);
    long long added = 0;
    GF_CUDA(cudaMemcpyAsync(&added, cnt, 8, cudaMemcpyDeviceToHost, s));
    GF_CUDA(cudaStreamSynchronize(s));
    t->count += added;
    return GF_OK;
  }
  // edge table: strictly increasing, above the current max (features.py:84-105)
  int* bad = reinterpret_cast<int*>(mm + 2);
  GF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  GF_LAUNCH(k_edge_check, grid_for(n, 256, G), 256, 0, s, d_ids, n, t->last_id, bad, mm);
  int hbad = 0;
  long long last = 0;
  GF_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaMemcpyAsync(&last, mm, 8, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  if (hbad) return fail(GF_EINVAL, "edge ids must be strictly increasing and exceed the current maximum");
  if (t->n + n > t->cap) {
    int64_t nc = std::max<int64_t>(t->n + n, std::max<int64_t>(64, 2 * t->cap));
    GF_TRY(grow(t->rows, t->n * t->pitch, nc * t->pitch, s));
    GF_TRY(grow(t->ids, t->n, nc, s));
    t->cap = nc;
  }
  GF_CUDA(cudaMemcpyAsync(t->ids + t->n, d_ids, 8 * n, cudaMemcpyDeviceToDevice, s));
  GF_LAUNCH(k_copy_rows_packed, grid_for(n * 32, 256, G), 256, 0, s, d_rows, n, t->dim, t->rows + t->n * t->pitch, t->pitch);
  GF_CUDA(cudaStreamSynchronize(s));
  t->n += n;
  t->last_id = last;
  return GF_OK;
}

gf_status gf_ftable_get(gf_ftable* t, const int64_t* d_ids, int64_t n, float* d_rows, uint8_t* d_found, void* stream) {
  if (!t) return fail(GF_EINVAL, "NULL argument");
  if (n == 0) return GF_OK;
  DeviceGuard dg(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sb(s);
  GF_TRY(sb.alloc((size_t)n * 8));
  int64_t* idx = sb.as<int64_t>();
  GF_TRY(ftable_get_idx(t, d_ids, n, idx, d_found, s));
  return gather(t->rows, t->pitch, idx, nullptr, n, t->dim, d_rows, t->dim, s);
}

gf_status gf_gather_rows(const float* d_table, int64_t ld, const int64_t* d_idx, int64_t n, int64_t dim, float* d_out,
                         void* stream) {
  if (n > 0 && (!d_table || !d_idx || !d_out)) return fail(GF_EINVAL, "NULL array");
  return gather(d_table, ld, d_idx, nullptr, n, dim, d_out, dim, (cudaStream_t)stream);
}



gf_status gf_fetch_features(gf_cache* c, gf_ftable* t, const int64_t* d_keys, int64_t n, float* d_values, uint8_t* d_hit,
                            int64_t* h_n_miss, int64_t* h_admitted, void* stream) {
  if (!c || !t || !h_n_miss || !h_admitted) return fail(GF_EINVAL, "NULL argument");
  if (t->dim != c->dim) return fail(GF_EINVAL, "cache and table dims differ");
  if (n > 0 && (!d_keys || !d_hit)) return fail(GF_EINVAL, "NULL array");
  *h_n_miss = 0;
  *h_admitted = 0;
  if (n == 0) return GF_OK;
  DeviceGuard dg(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t G = 8 * num_sms();
  const int64_t dim = c->dim, cap = c->capacity;
  const bool lru_lfu = c->policy != GF_CACHE_FIFO && c->max_update > 0;
  const int64_t ssize = pow2_at_least(2 * n);
  size_t scan_bytes = 0, free_bytes = 0;
  GF_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, scan_bytes, (longlong2*)nullptr, (longlong2*)nullptr, AddLL2(),
                                         make_longlong2(0, 0), (int)(n + 1), s));
  if (lru_lfu)
    GF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, free_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)(cap + 1), s));
  Scratch sb(s);
  int32_t* slots;
  int64_t *tidx, *okeys, *osrc, *sk, *ff = nullptr, *fpos = nullptr, *free_slots = nullptr;
  long long *smin, *mm = nullptr, *counts;
  uint8_t* found;
  longlong2 *flag2, *pos2;
  void *scan_tmp, *free_tmp = nullptr;
  float* values = d_values;
  auto carve = [&](Arena& a) {
    slots = a.take<int32_t>(n);
    tidx = a.take<int64_t>(n);
    found = a.take<uint8_t>(n);
    flag2 = a.take<longlong2>(n + 1);
    pos2 = a.take<longlong2>(n + 1);
    okeys = a.take<int64_t>(n);
    osrc = a.take<int64_t>(n);
    sk = a.take<int64_t>(ssize);
    smin = a.take<long long>(ssize);
    counts = a.take<long long>(8);
    scan_tmp = a.take<char>((int64_t)scan_bytes);
    if (lru_lfu) {
      ff = a.take<int64_t>(cap + 1);
      fpos = a.take<int64_t>(cap + 1);
      free_slots = a.take<int64_t>(cap + 1);
      mm = a.take<long long>(2);
      free_tmp = a.take<char>((int64_t)free_bytes);
    }
    if (!d_values) values = a.take<float>(n * dim);  // rows are still needed for the insert
  };
  {
    Arena probe;
    carve(probe);
    GF_TRY(sb.alloc(probe.off + 4096));
    Arena A;
    A.base = sb.as<char>();
    carve(A);
  }
  if (!c->hsmall) GF_CUDA(cudaMallocHost(&c->hsmall, 64));
  // cache.fetch(keys) (harness.py:438, cache.py:85-121): probe, score event, miss counting
  GF_LAUNCH(k_lookup, grid_for(n, 256, G), 256, 0, s, d_keys, n, c->hkeys, c->hslots, c->tsize - 1, slots, d_hit,
            c->counters);
  // store.get(miss) (harness.py:440): table row of every occurrence; hits and misses are then
  // copied to the output in one pass, each row once
  GF_TRY(ftable_get_idx(t, d_keys, n, tidx, found, s));
  GF_TRY(fetch_gather(c, slots, t, tidx, n, values, s));
  if (c->policy == GF_CACHE_LRU) {
    GF_LAUNCH(k_lru_decay, grid_for(cap, 256, G), 256, 0, s, c->keys, c->scores, cap);
    GF_LAUNCH(k_score_hits, grid_for(n, 256, G), 256, 0, s, slots, n, c->scores, 0);
  } else if (c->policy == GF_CACHE_LFU) {
    GF_LAUNCH(k_score_hits, grid_for(n, 256, G), 256, 0, s, slots, n, c->scores, 1);
  }
  GF_LAUNCH(k_count_misses, grid_for(n, 256, G), 256, 0, s, d_hit, (const int32_t*)nullptr, n, c->counters + 1);
  // free slots and the occupied score range, ahead of the placement (the fetch changes no key)
  if (lru_lfu) {
    GF_LAUNCH(k_mm_init, 1, 1, 0, s, mm);
    GF_LAUNCH(k_free_flags, grid_for(cap, 256, G), 256, 0, s, c->keys, c->scores, cap, ff, mm);
    size_t fb = free_bytes;
    GF_CUDA(cub::DeviceScan::ExclusiveSum(free_tmp, fb, ff, fpos, (int)(cap + 1), s));
    GF_LAUNCH(k_free_scatter, grid_for(cap, 256, G), 256, 0, s, ff, fpos, cap, free_slots);
  }
  // distinct misses (first-occurrence order) and the found ones among them, in one scan
  GF_CUDA(cudaMemsetAsync(sk, 0xff, (size_t)ssize * 8, s));    // EMPTY_KEY = -1
  GF_CUDA(cudaMemsetAsync(smin, 0x7f, (size_t)ssize * 8, s));  // large
  GF_LAUNCH(k_first_insert, grid_for(n, 256, G), 256, 0, s, d_keys, n, slots, sk, smin, ssize - 1);
  GF_LAUNCH(k_ff_flags, grid_for(n, 256, G), 256, 0, s, d_keys, n, slots, sk, smin, ssize - 1, found, flag2);
  size_t sbt = scan_bytes;
  GF_CUDA(cub::DeviceScan::ExclusiveScan(scan_tmp, sbt, flag2, pos2, AddLL2(), make_longlong2(0, 0), (int)(n + 1), s));
  GF_LAUNCH(k_ff_scatter, grid_for(n, 256, G), 256, 0, s, d_keys, n, flag2, pos2, okeys, osrc);
  GF_LAUNCH(k_ff_counts, 1, 1, 0, s, pos2, n, fpos, cap, mm, counts);
  GF_CUDA(cudaMemcpyAsync(c->hsmall, counts, 5 * sizeof(long long), cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));  // the block's one synchronisation
  const long long* hc = c->hsmall;
  *h_n_miss = hc[0];
  const int64_t nf = hc[1];
  if (nf == 0) return GF_OK;
  // insert_batch(miss[found], rows[found]) (harness.py:441): rows are read back from the output
  FreeState pre{free_slots, hc[2], hc[3], hc[4]};
  return place_impl(c, okeys, osrc, nf, values, h_admitted, s, &pre);
}

}  // extern "C"
