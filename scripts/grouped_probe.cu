// Probe: does processing uniform hop-1 queries grouped by node buy L2 line reuse, and what do the
// scattered (query-order) CSR writes cost?  GDELT-shaped pick stream (17K nodes, 191M slots, node
// weights i^-1/(skew-1), 10.5M queries, 10 picks each uniform over a prefix of the node's list).
//   mode A: query order, coalesced output (the fused kernel's pattern)
//   mode B: node-sorted order, outputs written at the query's own CSR position (random 80 B runs)
//   mode C: node-sorted order, outputs written in processing order (read-reuse bound)
// (mode A loads evict-first like the fused kernel; B and C load with the default policy so lines stay for reuse)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a grouped_probe.cu -o grouped_probe
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
#include <algorithm>
#include <cuda_runtime.h>

__host__ __device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31);
}
constexpr int BLK_SHIFT = 13;  // 8192-slot blocks scattered over the pool

__global__ void k_init(int64_t* rec, int64_t nslots) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslots; i += (int64_t)gridDim.x * blockDim.x) {
    rec[4 * i] = i; rec[4 * i + 1] = i * 3; rec[4 * i + 2] = i & 0xffff; rec[4 * i + 3] = 1;
  }
}
__global__ void k_queries(const double* cdf, int nn, const int64_t* deg, int64_t nq, uint32_t* qnode, int64_t* qn) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const double u = (mix(q * 2 + 1) >> 11) * (1.0 / 9007199254740992.0);
    int lo = 0, hi = nn - 1;
    while (lo < hi) { int m = (lo + hi) / 2; if (cdf[m] > u) hi = m; else lo = m + 1; }
    const double f = ((mix(q * 2 + 2) >> 11) + 1) * (1.0 / 9007199254740992.0);
    qnode[q] = lo;
    qn[q] = max((int64_t)1, (int64_t)(f * deg[lo]));
  }
}
template <int MODE>
__global__ void k_gather(const int64_t* __restrict__ rec, const int64_t* __restrict__ start, const int32_t* __restrict__ bmap,
                         const uint32_t* __restrict__ qnode, const int64_t* __restrict__ qn, const uint32_t* __restrict__ perm,
                         int64_t nq, int64_t* onbr, int64_t* oeid, int64_t* ots) {
  const int64_t ne = nq * 10;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qs = e / 10, i = e - qs * 10;
    const int64_t q = MODE == 0 ? qs : perm[qs];
    const uint32_t v = qnode[q];
    const int64_t n = qn[q];
    const int64_t p = (int64_t)(mix(q * 16 + i) % (uint64_t)n);
    const int64_t g = start[v] + p;
    const int64_t slot = ((int64_t)bmap[g >> BLK_SHIFT] << BLK_SHIFT) | (g & ((1 << BLK_SHIFT) - 1));
    long long x0, x1, x2, x3;
    if (MODE == 0)
      asm volatile("ld.global.nc.L2::evict_first.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(rec + 4 * slot));
    else
      asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(rec + 4 * slot));
    const int64_t at = MODE == 1 ? q * 10 + i : e;
    __stcs((long long*)onbr + at, x2);
    __stcs((long long*)oeid + at, x1);
    __stcs((long long*)ots + at, x0);
  }
}
int main() {
  const int nn = 17000;
  const int64_t E = 191000000, nq = 10500000;
  std::vector<double> w(nn), cdf(nn);
  double s = 0;
  for (int i = 0; i < nn; i++) { w[i] = std::pow(i + 1.0, -1.0 / 1.2); s += w[i]; }
  std::vector<int64_t> deg(nn), start(nn);
  int64_t tot = 0; double c = 0;
  for (int i = 0; i < nn; i++) {
    deg[i] = std::max<int64_t>(1, (int64_t)(E * w[i] / s)); start[i] = tot; tot += deg[i];
    c += w[i] / s; cdf[i] = c;
  }
  cdf[nn - 1] = 1.0;
  const int64_t nblk = (tot >> BLK_SHIFT) + 1, nslots = nblk << BLK_SHIFT;
  std::vector<int32_t> bmap(nblk);
  for (int64_t i = 0; i < nblk; i++) bmap[i] = (int32_t)i;
  for (int64_t i = nblk - 1; i > 0; i--) std::swap(bmap[i], bmap[mix(i) % (i + 1)]);
  printf("nodes %d slots %lld (%.2f GB records) top deg %lld\n", nn, (long long)tot, nslots * 32 / 1e9, (long long)deg[0]);
  int64_t *rec, *dstart, *ddeg, *qn, *onbr, *oeid, *ots; double* dcdf; int32_t* dbmap; uint32_t *qnode, *perm, *knode;
  cudaMalloc(&rec, nslots * 32); cudaMalloc(&dstart, nn * 8); cudaMalloc(&ddeg, nn * 8); cudaMalloc(&dcdf, nn * 8);
  cudaMalloc(&dbmap, nblk * 4); cudaMalloc(&qn, nq * 8); cudaMalloc(&qnode, nq * 4); cudaMalloc(&perm, nq * 4);
  cudaMalloc(&knode, nq * 4);
  cudaMalloc(&onbr, nq * 80); cudaMalloc(&oeid, nq * 80); cudaMalloc(&ots, nq * 80);
  cudaMemcpy(dstart, start.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ddeg, deg.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dcdf, cdf.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dbmap, bmap.data(), nblk * 4, cudaMemcpyHostToDevice);
  k_init<<<148 * 8, 256>>>(rec, nslots);
  k_queries<<<148 * 8, 256>>>(dcdf, nn, ddeg, nq, qnode, qn);
  // sort (node, query index): the grouping pass
  uint32_t* iota; cudaMalloc(&iota, nq * 4);
  std::vector<uint32_t> h(nq); for (int64_t i = 0; i < nq; i++) h[i] = (uint32_t)i;
  cudaMemcpy(iota, h.data(), nq * 4, cudaMemcpyHostToDevice);
  size_t tb = 0; void* tmp = nullptr;
  cub::DeviceRadixSort::SortPairs(tmp, tb, qnode, knode, iota, perm, (int)nq, 0, 15);
  cudaMalloc(&tmp, tb);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    cub::DeviceRadixSort::SortPairs(tmp, tb, qnode, knode, iota, perm, (int)nq, 0, 15);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("sort 10.5M (15-bit node, u32 index): %.3f ms\n", ms);
  for (int grid : {148 * 8, 148 * 16}) {
    for (int mode = 0; mode < 3; mode++) {
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        if (mode == 0) k_gather<0><<<grid, 256>>>(rec, dstart, dbmap, qnode, qn, perm, nq, onbr, oeid, ots);
        if (mode == 1) k_gather<1><<<grid, 256>>>(rec, dstart, dbmap, qnode, qn, perm, nq, onbr, oeid, ots);
        if (mode == 2) k_gather<2><<<grid, 256>>>(rec, dstart, dbmap, qnode, qn, perm, nq, onbr, oeid, ots);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("grid %d mode %c: %.3f ms  %.2f G picks/s\n", grid, "ABC"[mode], ms, nq * 10 / ms / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
