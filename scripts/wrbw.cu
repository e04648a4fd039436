// HBM write-bandwidth probe (B200): how fast can a kernel stream int64 outputs to HBM?
// Modes: three interleaved int64 streams with 8 B st.global.cs (the sampler's CSR stores),
// the same with default stores, 16 B vector stores, and a plain copy (read + write) for reference.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/wrbw scripts/wrbw.cu && scripts/wrbw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void w3_cs(long long* a, long long* b, long long* c, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    __stcs(a + i, (long long)i);
    __stcs(b + i, (long long)i * 3);
    __stcs(c + i, (long long)i * 7);
  }
}
__global__ void w3_wb(long long* a, long long* b, long long* c, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    a[i] = (long long)i;
    b[i] = (long long)i * 3;
    c[i] = (long long)i * 7;
  }
}
__global__ void w1_v4(int4* a, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    __stcs(a + i, make_int4((int)i, 1, 2, 3));
}
__global__ void copy_v4(const int4* __restrict__ s, int4* d, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    d[i] = __ldcs(s + i);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = 105ull << 20;  // 105M int64 per stream (the recent hop-1 output)
  long long *a, *b, *c;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMalloc(&c, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%-34s %8.3f ms  %8.1f GB/s\n", name, best, bytes / (best / 1e3) / 1e9);
  };
  for (int blocks : {sms * 4, sms * 8, sms * 16}) {
    printf("grid %d x 256\n", blocks);
    timeit("3 streams int64, st.global.cs", 3.0 * n * 8, [&] { w3_cs<<<blocks, 256>>>(a, b, c, n); });
    timeit("3 streams int64, st.global", 3.0 * n * 8, [&] { w3_wb<<<blocks, 256>>>(a, b, c, n); });
    timeit("1 stream 16 B st.global.cs", 3.0 * n * 8, [&] { w1_v4<<<blocks, 256>>>((int4*)a, 3 * n / 2); });
    timeit("copy 16 B (read+write bytes)", 2.0 * n * 8,
           [&] { copy_v4<<<blocks, 256>>>((const int4*)a, (int4*)b, n / 2); });
  }
  return 0;
}
