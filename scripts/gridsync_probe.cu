// Probe: cost of a cooperative-groups grid barrier and of a dependent L2 load chain on B200
// (the floor of the cooperative ingest kernel's phases).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a gridsync_probe.cu -o gridsync_probe
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; i++) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}
__global__ void k_chain(const int* __restrict__ next, int steps, int* sink) {
  int p = (blockIdx.x * blockDim.x + threadIdx.x) & 1023;
  for (int i = 0; i < steps; i++) p = __ldcg(next + p);
  if (p == -5) sink[1] = p;
}
int main() {
  int* sink; cudaMalloc(&sink, 64);
  int* next; cudaMalloc(&next, 1 << 24);
  int h[1 << 12]; for (int i = 0; i < 4096; i++) h[i] = (i * 977 + 13) & 4095;
  cudaMemcpy(next, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int T : {256, 512, 1024}) {
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sync, T, 0);
    for (int G : {16, 64, 148, 148 * 2}) {
      if (G > 148 * occ) continue;
      float ms[2];
      for (int rep = 0; rep < 3; rep++)
        for (int k = 0; k < 2; k++) {
          int iters = k ? 101 : 1;
          void* args[] = {&iters, &sink};
          cudaEventRecord(a);
          cudaLaunchCooperativeKernel((void*)k_sync, G, T, args, 0, 0);
          cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms[k], a, b);
        }
      printf("grid.sync  G=%4d T=%4d: %.2f us per barrier (launch+1 sync %.1f us)\n", G, T, (ms[1] - ms[0]) * 10.0, ms[0] * 1e3);
    }
  }
  for (int steps : {1, 101}) {
    float ms;
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a);
      k_chain<<<148, 256>>>(next, steps, sink);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    }
    printf("L2 chain steps=%d: %.2f us\n", steps, ms * 1e3);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
