// gf_part.cu -- device side of the multi-GPU exchanges.
//
// The reference routes work to the machine that owns it and merges the answers back in request
// order (cluster.py:242-292 per-hop sampling scatter/gather, cluster.py:296-325 feature fetch).
// Around each all-to-all (NCCL over NVLink; gloo in the CPU tests) this file provides:
//   gf_bucket_by_owner  stable counting sort of keys by owner = key mod P (partition.py:38-39 uses
//                       Python's floor modulo): per-CTA owner histograms, one exclusive scan in
//                       owner-major order, a stable in-CTA scatter -> the send order + P counts
//   gf_csr_merge        owner answers (per-query counts + flat edge arrays, bucketed order) back
//                       to the original query order: counts scattered, offsets scanned, each
//                       query's run copied to its CSR slot (cluster.py:268-292)
//   gf_scatter_rows     feature rows back to the original key order (out[dest[i]] = in[i]),
//                       128-bit copies when rows are 16-byte pitched
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "gf_common.cuh"

using namespace gf;

namespace {

constexpr int BT = 256, BI = 4, BTILE = BT * BI;  // bucketing: 1024 keys per CTA
constexpr int PMAX = 64;

__device__ __forceinline__ int owner_of(int64_t k, int P) {
  int64_t r = k % P;
  return (int)(r < 0 ? r + P : r);
}

// per-CTA owner histogram, written owner-major: hist[p * nct + cta]
__global__ void __launch_bounds__(BT) k_bucket_hist(const int64_t* __restrict__ keys, int64_t n, int P, int64_t nct,
                                                    int64_t* __restrict__ hist) {
  __shared__ int h[PMAX];
  for (int p = threadIdx.x; p < P; p += BT) h[p] = 0;
  __syncthreads();
  const int64_t i0 = blockIdx.x * (int64_t)BTILE;
#pragma unroll
  for (int j = 0; j < BI; j++) {
    const int64_t i = i0 + j * BT + threadIdx.x;
    if (i < n) atomicAdd(&h[owner_of(keys[i], P)], 1);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += BT) hist[p * nct + blockIdx.x] = h[p];
}

// stable scatter: within the CTA, keys keep their index order per owner (one block scan per owner)
__global__ void __launch_bounds__(BT) k_bucket_scatter(const int64_t* __restrict__ keys, int64_t n, int P, int64_t nct,
                                                       const int64_t* __restrict__ off, int64_t* __restrict__ perm,
                                                       int64_t* __restrict__ keys_out, int64_t* __restrict__ counts) {
  typedef cub::BlockScan<int, BT> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const int64_t i0 = blockIdx.x * (int64_t)BTILE + (int64_t)threadIdx.x * BI;  // blocked: thread owns BI keys
  int64_t k[BI];
  int ow[BI];
#pragma unroll
  for (int j = 0; j < BI; j++) {
    const int64_t i = i0 + j;
    k[j] = i < n ? keys[i] : 0;
    ow[j] = i < n ? owner_of(k[j], P) : -1;
  }
  for (int p = 0; p < P; p++) {
    int f[BI], s[BI];
#pragma unroll
    for (int j = 0; j < BI; j++) f[j] = ow[j] == p;
    Scan(tmp).ExclusiveSum(f, s);
    __syncthreads();
    const int64_t base = off[p * nct + blockIdx.x];
#pragma unroll
    for (int j = 0; j < BI; j++)
      if (f[j]) {
        perm[base + s[j]] = i0 + j;
        if (keys_out) keys_out[base + s[j]] = k[j];
      }
  }
  if (blockIdx.x == 0)  // owner totals from the owner-major scan (off[P * nct] = n)
    for (int p = threadIdx.x; p < P; p += BT) counts[p] = off[(p + 1) * nct] - off[p * nct];
}

__global__ void k_scatter_counts(const int64_t* __restrict__ perm, const int64_t* __restrict__ cnt, int64_t n,
                                 int64_t* __restrict__ cnt_orig) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    cnt_orig[perm[i]] = cnt[i];
}

struct Arrs {
  const int64_t* in[8];
  int64_t* out[8];
  int k;
};

// one thread per bucketed query: its run [start[i], +cnt[i]) goes to [offsets[perm[i]], ...)
__global__ void k_merge_runs(const int64_t* __restrict__ perm, const int64_t* __restrict__ cnt,
                             const int64_t* __restrict__ start, const int64_t* __restrict__ offsets, int64_t n, Arrs A) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cnt[i], s = start[i], d = offsets[perm[i]];
    for (int a = 0; a < A.k; a++)
      for (int64_t j = 0; j < c; j++) A.out[a][d + j] = A.in[a][s + j];
  }
}

__global__ void k_scatter_rows(const float* __restrict__ in, int64_t ld_in, const int64_t* __restrict__ dest, int64_t n,
                               int64_t dim, float* __restrict__ out, int64_t ld_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = ((ld_in | ld_out | dim) & 3) == 0 && ((((uintptr_t)in) | ((uintptr_t)out)) & 15) == 0;
  for (int64_t i = warp; i < n; i += nw) {
    const float* src = in + i * ld_in;
    float* dst = out + dest[i] * ld_out;
    if (vec) {
      for (int64_t c = lane; c < dim / 4; c += 32)
        reinterpret_cast<float4*>(dst)[c] = __ldg(reinterpret_cast<const float4*>(src) + c);
    } else {
      for (int64_t c = lane; c < dim; c += 32) dst[c] = __ldg(src + c);
    }
  }
}

}  // namespace

extern "C" {

gf_status gf_bucket_by_owner(const int64_t* d_keys, int64_t n, int nparts, int64_t* d_perm, int64_t* d_keys_out,
                             int64_t* h_counts, void* stream) {
  if (nparts < 1 || nparts > PMAX) return fail(GF_EINVAL, "nparts must be in [1, 64]");
  if (n < 0 || (n > 0 && (!d_keys || !d_perm)) || !h_counts) return fail(GF_EINVAL, "NULL argument");
  for (int p = 0; p < nparts; p++) h_counts[p] = 0;
  if (n == 0) return GF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nct = (n + BTILE - 1) / BTILE, H = nparts * nct + 1;
  size_t scan_bytes = 0;
  GF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)H, s));
  Scratch sb(s);
  GF_TRY(sb.alloc(sizeof(int64_t) * (2 * H + PMAX) + scan_bytes + 256));
  int64_t* hist = sb.as<int64_t>();
  int64_t* off = hist + H;
  int64_t* cnt = off + H;
  void* tmp = cnt + PMAX;
  GF_CUDA(cudaMemsetAsync(hist + H - 1, 0, sizeof(int64_t), s));  // the scan's last entry = n
  GF_LAUNCH(k_bucket_hist, nct, BT, 0, s, d_keys, n, nparts, nct, hist);
  GF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, hist, off, (int)H, s));
  GF_LAUNCH(k_bucket_scatter, nct, BT, 0, s, d_keys, n, nparts, nct, off, d_perm, d_keys_out, cnt);
  GF_CUDA(cudaMemcpyAsync(h_counts, cnt, sizeof(int64_t) * nparts, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_csr_merge(const int64_t* d_perm, const int64_t* d_cnt_sorted, int64_t n, int narr,
                       const int64_t* const* d_in, int64_t* d_offsets, int64_t* const* d_out, int64_t* h_total,
                       void* stream) {
  if (narr < 0 || narr > 8) return fail(GF_EINVAL, "at most 8 edge arrays");
  if (!d_offsets || !h_total || (n > 0 && (!d_perm || !d_cnt_sorted))) return fail(GF_EINVAL, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  *h_total = 0;
  if (n == 0) {
    GF_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), s));
    GF_CUDA(cudaStreamSynchronize(s));
    return GF_OK;
  }
  size_t scan_bytes = 0;
  GF_CUDA(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)n, s));
  Scratch sb(s);
  GF_TRY(sb.alloc(sizeof(int64_t) * (2 * n + 2) + scan_bytes + 256));
  int64_t* cnt_orig = sb.as<int64_t>();
  int64_t* start = cnt_orig + n;  // [n + 1]: exclusive prefix of the bucketed counts
  void* tmp = start + n + 2;
  const int64_t G = 8 * num_sms();
  GF_LAUNCH(k_scatter_counts, grid_for(n, 256, G), 256, 0, s, d_perm, d_cnt_sorted, n, cnt_orig);
  GF_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), s));
  GF_CUDA(cub::DeviceScan::InclusiveSum(tmp, scan_bytes, cnt_orig, d_offsets + 1, (int)n, s));
  GF_CUDA(cudaMemsetAsync(start, 0, sizeof(int64_t), s));
  GF_CUDA(cub::DeviceScan::InclusiveSum(tmp, scan_bytes, d_cnt_sorted, start + 1, (int)n, s));
  Arrs A{};
  A.k = narr;
  for (int a = 0; a < narr; a++) {
    A.in[a] = d_in[a];
    A.out[a] = d_out[a];
  }
  if (narr > 0) GF_LAUNCH(k_merge_runs, grid_for(n, 256, G), 256, 0, s, d_perm, d_cnt_sorted, start, d_offsets, n, A);
  GF_CUDA(cudaMemcpyAsync(h_total, d_offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

gf_status gf_scatter_rows(const float* d_in, int64_t ld_in, const int64_t* d_dest, int64_t n, int64_t dim, float* d_out,
                          int64_t ld_out, void* stream) {
  if (n > 0 && (!d_in || !d_dest || !d_out)) return fail(GF_EINVAL, "NULL argument");
  if (n <= 0 || dim <= 0) return GF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  GF_LAUNCH(k_scatter_rows, std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 32), 256, 0, s, d_in, ld_in, d_dest, n,
            dim, d_out, ld_out);
  return GF_OK;
}

}  // extern "C"
