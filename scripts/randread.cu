// Microbenchmark: random 32-byte record gathers from a large HBM array (design probe for the
// uniform-sampling write pass).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a randread.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31);
}
template <int MODE>
__global__ void gather(const int4* __restrict__ a, int64_t nrec, int64_t n, long long* out) {
  long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = mix(i) % nrec;
    const int4* p = a + 2 * r;
    int4 x, y;
    if (MODE == 0) { x = __ldg(p); y = __ldg(p + 1); }
    else if (MODE == 1) {
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(p));
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(y.x), "=r"(y.y), "=r"(y.z), "=r"(y.w) : "l"(p + 1));
    } else if (MODE == 2) { x = __ldcs(p); y = __ldcs(p + 1); }
    else { x = __ldg(p); y = make_int4(0,0,0,0); }
    acc += x.x + x.w + y.x + y.z;
  }
  if (acc == 42) *out = acc;
}
int main() {
  int64_t nrec = (int64_t)7 << 27;  // 7*128M*32B = 28.7 GB? keep 7.5 GB
  nrec = 240000000;                 // 7.7 GB
  int4* a; cudaMalloc(&a, nrec * 32); cudaMemset(a, 1, nrec * 32);
  long long* o; cudaMalloc(&o, 8);
  int64_t n = 200000000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int gran : {128, 64, 32}) {
  cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
  size_t got = 0; cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
  printf("L2 fetch granularity %d (reads back %zu)\n", gran, got);
  for (int mode = 0; mode < 4; mode++) {
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      if (mode == 0) gather<0><<<148 * 16, 256>>>(a, nrec, n, o);
      if (mode == 1) gather<1><<<148 * 16, 256>>>(a, nrec, n, o);
      if (mode == 2) gather<2><<<148 * 16, 256>>>(a, nrec, n, o);
      if (mode == 3) gather<3><<<148 * 16, 256>>>(a, nrec, n, o);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("mode %d: %.3f ms  %.2f G records/s  (%.1f GB/s of 32B records)\n", mode, ms, n / ms / 1e6, n * 32.0 / ms / 1e6);
    }
  }
  }
  return 0;
}
