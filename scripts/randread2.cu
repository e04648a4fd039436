// Random 32-byte record gathers: which load flavour moves the fewest DRAM bytes per record?
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a randread2.cu -o randread2
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
    const int64_t r = mix(i) % nrec;
    const void* p = a + 2 * r;
    long long x0, x1, x2, x3;
    if (MODE == 0) asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(p));
    if (MODE == 1) asm volatile("ld.global.cg.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(p));
    if (MODE == 2) asm volatile("ld.global.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(p));
    if (MODE == 3) asm volatile("ld.global.cv.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(p));
    if (MODE == 4) asm volatile("ld.global.nc.L2::64B.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(p));
    if (MODE == 5) asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(p));
    if (MODE == 6) { asm volatile("ld.global.cg.v2.b64 {%0,%1}, [%2];" : "=l"(x0), "=l"(x1) : "l"(p)); x2 = x3 = 0; }
    acc += x0 ^ x1 ^ x2 ^ x3;
  }
  if (acc == 42) *out = acc;
}
int main() {
  const int64_t nrec = 240000000;  // 7.7 GB
  int4* a; cudaMalloc(&a, nrec * 32); cudaMemset(a, 1, nrec * 32);
  long long* o; cudaMalloc(&o, 8);
  const int64_t n = 200000000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int gran : {0, 32}) {
    if (gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    for (int mode = 0; mode < 7; mode++) {
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        switch (mode) {
          case 0: gather<0><<<148 * 16, 256>>>(a, nrec, n, o); break;
          case 1: gather<1><<<148 * 16, 256>>>(a, nrec, n, o); break;
          case 2: gather<2><<<148 * 16, 256>>>(a, nrec, n, o); break;
          case 3: gather<3><<<148 * 16, 256>>>(a, nrec, n, o); break;
          case 4: gather<4><<<148 * 16, 256>>>(a, nrec, n, o); break;
          case 5: gather<5><<<148 * 16, 256>>>(a, nrec, n, o); break;
          case 6: gather<6><<<148 * 16, 256>>>(a, nrec, n, o); break;
        }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("gran %d mode %d: %.3f ms  %.2f G records/s\n", gran, mode, ms, n / ms / 1e6);
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
