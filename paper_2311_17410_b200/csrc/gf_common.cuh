// gf_common.cuh -- shared definitions for libgfb200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <atomic>
#include <string>

#include "../../include/gfb200.h"

#define GF_TS_MIN ((int64_t)(-9223372036854775807LL - 1))
#define GF_NO_BLOCK (-1LL)
#define GF_EMPTY_KEY (-1LL)
#define GF_PHILOX_TAG 0x47464232u  // "GFB2"

namespace gf {

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string& msg);
gf_status fail(gf_status st, const std::string& msg);
extern std::atomic<uint64_t> g_launches;
uint64_t seed_sequence_2(uint64_t a, uint64_t b);

#define GF_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      return ::gf::fail(GF_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define GF_TRY(expr)              \
  do {                            \
    gf_status _s = (expr);        \
    if (_s != GF_OK) return _s;   \
  } while (0)

// optional per-launch CUDA-event profiling (gf_profile_enable)
extern std::atomic<int> g_profile;
extern thread_local std::string g_prof_tag;  // appended to profiled kernel names
cudaEvent_t prof_start(cudaStream_t s);
void prof_stop(const char* name, cudaStream_t s, cudaEvent_t e0);

// launch + count + (optional) profile + check
#define GF_LAUNCH(kernel, grid, block, smem, stream, ...)                        \
  do {                                                                           \
    if ((grid) > 0) {                                                            \
      cudaEvent_t _gf_e0 = nullptr;                                              \
      if (::gf::g_profile.load(std::memory_order_relaxed))                       \
        _gf_e0 = ::gf::prof_start(stream);                                       \
      kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                \
      ::gf::g_launches.fetch_add(1, std::memory_order_relaxed);                  \
      if (_gf_e0) ::gf::prof_stop(#kernel, stream, _gf_e0);                      \
      GF_CUDA(cudaGetLastError());                                               \
    }                                                                            \
  } while (0)

// Programmatic dependent launch (PDL) for dependent kernel sequences (the ingest graph): a kernel
// launched with GF_LAUNCH_PDL may start while its predecessor is still running; it calls
// gf::pdl_enter() first, which lets its own successor launch early and then waits until the
// predecessor grid has completed and its writes are visible (griddepcontrol; a no-op for
// kernels launched without the attribute).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

#define GF_LAUNCH_PDL(kernel, grid, block, smem, strm_, ...)                                     \
  do {                                                                                            \
    if ((grid) > 0) {                                                                             \
      cudaEvent_t _gf_e0 = nullptr;                                                               \
      if (::gf::g_profile.load(std::memory_order_relaxed)) _gf_e0 = ::gf::prof_start(strm_);     \
      cudaLaunchConfig_t _gf_cfg = {};                                                            \
      cudaLaunchAttribute _gf_attr[1];                                                            \
      _gf_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                        \
      _gf_attr[0].val.programmaticStreamSerializationAllowed = 1;                                 \
      _gf_cfg.gridDim = dim3((unsigned)(grid));                                                   \
      _gf_cfg.blockDim = dim3((unsigned)(block));                                                 \
      _gf_cfg.dynamicSmemBytes = (smem);                                                          \
      _gf_cfg.stream = (strm_);                                                                  \
      _gf_cfg.attrs = _gf_attr;                                                                   \
      _gf_cfg.numAttrs = 1;                                                                       \
      GF_CUDA(cudaLaunchKernelEx(&_gf_cfg, kernel, __VA_ARGS__));                                 \
      ::gf::g_launches.fetch_add(1, std::memory_order_relaxed);                                   \
      if (_gf_e0) ::gf::prof_stop(#kernel, strm_, _gf_e0);                                       \
    }                                                                                             \
  } while (0)

inline void init_device_pool(int dev);

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
    init_device_pool(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

// Keep freed stream-ordered scratch mapped (the default pool would return it to
// the OS at every synchronise, making each per-call cudaMallocAsync a remap).
inline void init_device_pool(int dev) {
  static std::atomic<uint64_t> done{0};
  uint64_t bit = 1ull << (dev & 63);
  if (done.load() & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (const char* g = getenv("GF_L2_FETCH_GRANULARITY")) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, atoi(g));
  done.fetch_or(bit);
}

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline int64_t grid_for(int64_t items, int per_block, int64_t cap_blocks = 0) {
  int64_t g = (items + per_block - 1) / per_block;
  if (cap_blocks > 0 && g > cap_blocks) g = cap_blocks;
  return g;
}

// stream-ordered scratch allocation
struct Scratch {
  cudaStream_t s;
  void* p = nullptr;
  size_t bytes = 0;
  explicit Scratch(cudaStream_t st) : s(st) {}
  gf_status alloc(size_t b) {
    release();
    bytes = b ? b : 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
      p = nullptr;
      return fail(GF_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    }
    return GF_OK;
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
  ~Scratch() { release(); }
};

// carve many small typed arrays out of one allocation
struct Arena {
  char* base = nullptr;
  size_t off = 0;
  template <class T>
  T* take(int64_t n) {
    off = (off + 255) & ~size_t(255);
    T* r = reinterpret_cast<T*>(base + off);
    off += sizeof(T) * (size_t)(n > 0 ? n : 1);
    return r;
  }
};

// ---- one edge slot (32 B, sector aligned) ----------------------------------
// ts/eid/nbr mirror SharedTier's neighbors/edge_ids/timestamps/valid
// (storage.py:201-217); owner lets a flat slot scan find the list it lives in.
struct __align__(32) Slot {
  int64_t ts;
  int64_t eid;
  int32_t nbr;
  int32_t owner;
  uint32_t valid;
  uint32_t pad;
};
static_assert(sizeof(Slot) == 32, "slot record must be one 32-byte sector");

// ---- RNG --------------------------------------------------------------------
__host__ __device__ inline void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
#else
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// d-th 64-bit draw of the stream keyed by (seed, qkey)
__host__ __device__ inline uint64_t rand64(uint64_t seed, uint64_t qkey, uint64_t d) {
  uint32_t c[4] = {(uint32_t)(d >> 1), (uint32_t)qkey, (uint32_t)(qkey >> 32), GF_PHILOX_TAG};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  return (d & 1) ? ((uint64_t)c[2] | ((uint64_t)c[3] << 32)) : ((uint64_t)c[0] | ((uint64_t)c[1] << 32));
}

__host__ __device__ inline uint64_t bounded64(uint64_t r, uint64_t range) {
#ifdef __CUDA_ARCH__
  return __umul64hi(r, range);
#else
  return (uint64_t)(((unsigned __int128)r * range) >> 64);
#endif
}

__host__ __device__ inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t child_key(uint64_t parent, uint64_t j) {
  return splitmix64(parent ^ (0x9E3779B97F4A7C15ull * (j + 1)));
}

// ---- cache-policy loads (sm_100a) ------------------------------------------------
#ifdef __CUDACC__
// one 256-bit load marked evict-first (random slot records, streaming windows); p 32-byte aligned
__device__ __forceinline__ void ld256_stream(const void* p, int64_t& a, int64_t& b, int64_t& c, int64_t& d) {
  asm volatile("ld.global.nc.L2::evict_first.v4.b64 {%0,%1,%2,%3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p));
}
#endif

// ---- warp helpers -----------------------------------------------------------
#ifdef __CUDACC__
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Number of elements < x in the non-decreasing sequence a[0], a[stride], ...
// a[(n-1)*stride]: 32-ary warp-ballot search, galloping at the tail first.
// All 32 lanes must call with identical arguments.
__device__ __forceinline__ int64_t warp_lower_bound(const int64_t* __restrict__ a, int stride, int64_t n,
                                                    int64_t x) {
  const int lane = lane_id();
  int64_t lo = 0, hi = n;
  if (n > 32) {
    int64_t p = n - 32 + lane;
    unsigned m = __ballot_sync(0xffffffffu, __ldg(a + p * stride) < x);
    if (m & 1u) return n - 32 + __popc(m);
    hi = n - 32;
  }
  while (hi - lo > 32) {
    int64_t step = (hi - lo + 31) / 32;
    int64_t p = lo + lane * step;
    bool lt = (p < hi) && (__ldg(a + p * stride) < x);
    int c = __popc(__ballot_sync(0xffffffffu, lt));
    if (c == 0) return lo;
    int64_t plast = lo + (int64_t)(c - 1) * step;
    int64_t nh = plast + step;
    lo = plast + 1;
    if (nh < hi) hi = nh;
  }
  int64_t p = lo + lane;
  bool lt = (p < hi) && (__ldg(a + p * stride) < x);
  return lo + __popc(__ballot_sync(0xffffffffu, lt));
}

// per-thread binary search: number of elements <= x in a[0..n)
__device__ __forceinline__ int64_t upper_bound_seq(const int64_t* __restrict__ a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (__ldg(a + m) <= x) lo = m + 1;
    else hi = m;
  }
  return lo;
}
#endif

}  // namespace gf
