// L2 read bandwidth probe (B200): every SM streams repeatedly over a buffer that fits in L2, with
// 128-bit loads, after a warm-up pass; reports the best GB/s over buffer sizes 8..64 MB.
// Writes profiles/l2_bandwidth.json (used by bench.py for L2-resident configs).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/l2bw scripts/l2bw.cu && scripts/l2bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const int4* __restrict__ p, size_t n, int reps, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; r++) {
    // each CTA starts at a different offset so the passes do not march in lock step
    for (size_t i = (blockIdx.x * blockDim.x + threadIdx.x + (size_t)r * 4099 * blockDim.x) % n, c = 0; c < n / stride;
         c++, i = (i + stride) % n) {
      int4 v = __ldcg(p + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double best = 0;
  size_t best_mb = 0;
  FILE* f = fopen("profiles/l2_bandwidth.json", "w");
  for (size_t mb : {8, 16, 32, 48, 64}) {
    size_t bytes = mb << 20, n = bytes / 16;
    int4 *p, *sink;
    cudaMalloc(&p, bytes);
    cudaMalloc(&sink, 64);
    cudaMemset(p, 1, bytes);
    const int reps = 20;
    rd<<<sms * 4, 512>>>(p, n, 2, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    rd<<<sms * 4, 512>>>(p, n, reps, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const size_t stride = (size_t)sms * 4 * 512;
    double moved = (double)(n / stride) * stride * 16 * reps;
    double gbs = moved / (ms / 1e3) / 1e9;
    printf("%zu MB: %.1f GB/s\n", mb, gbs);
    if (gbs > best) best = gbs, best_mb = mb;
    cudaFree(p);
    cudaFree(sink);
  }
  if (f) {
    fprintf(f, "{\"l2_read_gbs\": %.1f, \"buffer_mb\": %zu, \"how\": \"scripts/l2bw.cu: %d SMs x 4 CTAs x 512 threads, "
               "ld.global.cg 128-bit over an L2-resident buffer, 20 passes after a warm-up, best of 8..64 MB\"}\n",
            best, best_mb, sms);
    fclose(f);
  }
  return 0;
}
