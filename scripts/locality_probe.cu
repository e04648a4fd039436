// Probe kernels for scripts/locality_probe.py: gather 32-byte records by index and store three int64
// output columns, either at the element's own position (output order) or at a permuted position
// (node-grouped processing order, per-query runs scattered back to output order).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o scripts/locality_probe.so scripts/locality_probe.cu
#include <cstdint>
#include <cuda_runtime.h>

struct __align__(32) Rec { int64_t a, b, c, d; };

__device__ __forceinline__ Rec ld_rec(const Rec* p) {
  Rec r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0,%1,%2,%3}, [%4];"
               : "=l"(r.a), "=l"(r.b), "=l"(r.c), "=l"(r.d) : "l"(p));
  return r;
}

template <bool PERM>
__global__ void __launch_bounds__(256) k_gather(const Rec* __restrict__ rec, const int64_t* __restrict__ idx,
                                                const int64_t* __restrict__ perm, int64_t n, int64_t* o0, int64_t* o1,
                                                int64_t* o2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x * 2 + threadIdx.x; i < n; i += stride) {
    const int64_t i1 = i + blockDim.x;
    Rec r0 = ld_rec(rec + idx[i]);
    Rec r1;
    if (i1 < n) r1 = ld_rec(rec + idx[i1]);
    const int64_t e0 = PERM ? perm[i] : i;
    __stcs(o0 + e0, r0.a); __stcs(o1 + e0, r0.b); __stcs(o2 + e0, r0.c);
    if (i1 < n) {
      const int64_t e1 = PERM ? perm[i1] : i1;
      __stcs(o0 + e1, r1.a); __stcs(o1 + e1, r1.b); __stcs(o2 + e1, r1.c);
    }
  }
}

extern "C" float probe_gather(const void* rec, const int64_t* idx, const int64_t* perm, int64_t n, int64_t* o0,
                              int64_t* o1, int64_t* o2, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = 148 * 8;
  float best = 1e30f;
  void* flush;
  cudaMalloc(&flush, 512u << 20);
  for (int r = 0; r < reps; r++) {
    cudaMemset(flush, r, 512u << 20);
    cudaEventRecord(a);
    if (perm) k_gather<true><<<grid, 256>>>((const Rec*)rec, idx, perm, n, o0, o1, o2);
    else k_gather<false><<<grid, 256>>>((const Rec*)rec, idx, nullptr, n, o0, o1, o2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaFree(flush);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}
