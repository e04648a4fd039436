// gf_offload.cu -- DynamicGraph.offload_before on the device (reference storage.py:516-574, TGOF format
// storage.py:42-43, 535-556, parse_offload :624-647).
//
// Three stream-ordered steps, each recomputed from the same cutoff so the
// host can write the blob before anything changes (the reference assembles
// the whole file before unlinking, so an I/O failure leaves the graph intact):
//   plan   -- per node, the prefix of head-side blocks with tmax < cutoff and
//             size > 0; its blob bytes (12 per block header + 25 per slot)
//   write  -- the TGOF blob, node-major, blocks head->tail, slots in order
//   commit -- unlink the prefixes: head/tail/num_blocks/live degree, the
//             block directory start, NodeRec, slot validity (offloaded slots
//             are no longer part of any list) and the freed handles, which are
//             returned to the host free list in the reference's order.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "gf_graph.cuh"

using namespace gf;

namespace {

struct OffPlan {
  int64_t* nblk;   // prefix blocks per node
  int64_t* bytes;  // blob bytes per node (num_nodes + 1, scanned in place later)
  int64_t* edges;  // offloaded slots per node
};

__global__ void k_off_plan(int64_t num_nodes, const int64_t* __restrict__ head, const int64_t* __restrict__ bnext,
                           const int64_t* __restrict__ btmax, const int64_t* __restrict__ bsize, int64_t cutoff,
                           OffPlan P) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < num_nodes; v += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = 0, bytes = 0, edges = 0;
    for (int64_t h = head[v]; h != GF_NO_BLOCK && btmax[h] < cutoff && bsize[h] > 0; h = bnext[h]) {  // storage.py:529
      k++;
      bytes += 12 + 25 * bsize[h];
      edges += bsize[h];
    }
    P.nblk[v] = k;
    P.bytes[v] = bytes;
    P.edges[v] = edges;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    P.nblk[num_nodes] = 0;
    P.bytes[num_nodes] = 0;
    P.edges[num_nodes] = 0;
  }
}

__device__ __forceinline__ void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; i++) p[i] = (uint8_t)(v >> (8 * i));
}

// warp per node: block headers "<QI" (node, size), slots "<QQqB" (nbr, eid, ts, valid)
__global__ void k_off_write(int64_t num_nodes, const int64_t* __restrict__ nblk, const int64_t* __restrict__ boff,
                            const int64_t* __restrict__ head, const int64_t* __restrict__ bnext,
                            const int64_t* __restrict__ bsize, const int64_t* __restrict__ bbase, const Slot* __restrict__ slots,
                            uint8_t* blob) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < num_nodes; v += nw) {
    int64_t k = nblk[v];
    if (!k) continue;
    uint8_t* p = blob + boff[v];
    int64_t h = head[v];
    for (int64_t b = 0; b < k; b++) {
      int64_t sz = bsize[h], base = bbase[h];
      if (lane == 0) {
        put_le(p, (uint64_t)v, 8);
        put_le(p + 8, (uint64_t)sz, 4);
      }
      for (int64_t i = lane; i < sz; i += 32) {
        Slot s = slots[base + i];
        uint8_t* r = p + 12 + 25 * i;
        put_le(r, (uint64_t)(int64_t)s.nbr, 8);
        put_le(r + 8, (uint64_t)s.eid, 8);
        put_le(r + 16, (uint64_t)s.ts, 8);
        r[24] = s.valid ? 1 : 0;
      }
      p += 12 + 25 * sz;
      h = bnext[h];
    }
  }
}

struct OffCommit {
  int64_t *head, *tail, *num_blocks, *degree, *dir_off, *dir_cap;
  const int64_t* nslots;
  const uint8_t* node_valid;
  uint8_t* nflags;
  int64_t* nrec;
  int64_t *bnext, *bprev, *bsize, *bbase, *btmin;
  const int64_t* dir;
  Slot* slots;
  int64_t* freed;  // handles, node-major, at the scanned block offsets
};

__global__ void k_off_commit(int64_t num_nodes, const int64_t* __restrict__ nblk, const int64_t* __restrict__ hoff,
                             OffCommit C) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < num_nodes; v += nw) {
    const int64_t k = nblk[v];
    if (!k) continue;
    int64_t h = C.head[v], live = 0;
    for (int64_t b = 0; b < k; b++) {
      const int64_t sz = C.bsize[h], base = C.bbase[h];
      for (int64_t i = lane; i < sz; i += 32) {  // live degree drops by the valid slots (storage.py:563,573)
        live += C.slots[base + i].valid != 0;
        C.slots[base + i].valid = 0;
      }
      if (lane == 0) C.freed[hoff[v] + b] = h;  // free_block in list order (storage.py:564)
      h = C.bnext[h];
    }
    for (int o = 16; o; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
    if (lane == 0) {
      const int64_t new_head = h;  // next of the last offloaded block (storage.py:566)
      C.head[v] = new_head;
      if (new_head == GF_NO_BLOCK) C.tail[v] = GF_NO_BLOCK;
      else C.bprev[new_head] = GF_NO_BLOCK;
      const int64_t nb = C.num_blocks[v] - k;
      C.num_blocks[v] = nb;
      C.degree[v] -= live;
      C.dir_off[v] += k;  // directory keeps absolute list positions; it now starts at the new head
      C.dir_cap[v] -= k;
      C.nflags[v] |= 1;   // positions no longer follow the sizing law's closed form from 0
      int64_t* r = C.nrec + v * NREC;
      r[0] = C.dir_off[v];
      r[2] = nb | (C.node_valid[v] ? NREC_VALID : 0) | NREC_IRREG;
      if (nb > 0) {
        r[3] = C.dir[C.dir_off[v] * DIRW + 1];
        r[8] = C.dir[C.dir_off[v] * DIRW];
      }
    }
  }
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

}  // namespace

extern "C" {

gf_status gf_graph_offload_before(gf_graph* g, int64_t cutoff, uint8_t* h_blob, int64_t blob_cap, int64_t* h_blob_len,
                                  int64_t* h_edges, int commit, void* stream) {
  if (!g) return fail(GF_EINVAL, "graph is NULL");
  DeviceGuard dg(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = g->num_nodes;
  const int64_t hdr = 8;  // "TGOF" + u32 version
  if (h_blob_len) *h_blob_len = hdr;
  if (h_edges) *h_edges = 0;
  if (n == 0) {
    if (h_blob && blob_cap >= hdr) {
      memcpy(h_blob, "TGOF", 4);
      uint32_t ver = 1;
      memcpy(h_blob + 4, &ver, 4);
    }
    return GF_OK;
  }
  Scratch sb(s);
  Arena A;
  GF_TRY(sb.alloc((size_t)(n + 1) * 8 * 6 + 4096));
  A.base = sb.as<char>();
  OffPlan P{A.take<int64_t>(n + 1), A.take<int64_t>(n + 1), A.take<int64_t>(n + 1)};
  int64_t* boff = A.take<int64_t>(n + 1);
  int64_t* hoff = A.take<int64_t>(n + 1);
  int64_t* eoff = A.take<int64_t>(n + 1);
  const int64_t G = 8 * num_sms();
  GF_LAUNCH(k_off_plan, grid_for(n, 256, G), 256, 0, s, n, g->head, g->bnext, g->btmax, g->bsize, cutoff, P);
  GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, P.bytes, boff, (int)(n + 1), s); }, s));
  GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, P.nblk, hoff, (int)(n + 1), s); }, s));
  GF_TRY(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, P.edges, eoff, (int)(n + 1), s); }, s));
  int64_t tot[3];
  GF_CUDA(cudaMemcpyAsync(&tot[0], boff + n, 8, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaMemcpyAsync(&tot[1], hoff + n, 8, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaMemcpyAsync(&tot[2], eoff + n, 8, cudaMemcpyDeviceToHost, s));
  GF_CUDA(cudaStreamSynchronize(s));
  if (h_blob_len) *h_blob_len = hdr + tot[0];
  if (h_edges) *h_edges = tot[2];
  if (h_blob) {
    if (blob_cap < hdr + tot[0]) return fail(GF_ERANGE, "offload blob buffer too small");
    memcpy(h_blob, "TGOF", 4);  // storage.py:536-537
    uint32_t ver = 1;
    memcpy(h_blob + 4, &ver, 4);
    if (tot[0] > 0) {
      Scratch bb(s);
      GF_TRY(bb.alloc((size_t)tot[0]));
      GF_LAUNCH(k_off_write, grid_for(n * 32, 256, G), 256, 0, s, n, P.nblk, boff, g->head, g->bnext, g->bsize, g->bbase,
                g->slots, bb.as<uint8_t>());
      GF_CUDA(cudaMemcpyAsync(h_blob + hdr, bb.p, (size_t)tot[0], cudaMemcpyDeviceToHost, s));
      GF_CUDA(cudaStreamSynchronize(s));
    }
  }
  if (commit && tot[1] > 0) {
    Scratch fb(s);
    GF_TRY(fb.alloc((size_t)tot[1] * 8));
    OffCommit C{g->head, g->tail, g->num_blocks, g->degree, g->dir_off, g->dir_cap, g->nslots, g->node_valid, g->nflags,
                g->nrec, g->bnext, g->bprev, g->bsize, g->bbase, g->btmin, g->dir, g->slots, fb.as<int64_t>()};
    GF_LAUNCH(k_off_commit, grid_for(n * 32, 256, G), 256, 0, s, n, P.nblk, hoff, C);
    std::vector<int64_t> freed(tot[1]);
    GF_CUDA(cudaMemcpyAsync(freed.data(), fb.p, 8 * (size_t)tot[1], cudaMemcpyDeviceToHost, s));
    GF_CUDA(cudaStreamSynchronize(s));
    g->free_handles.insert(g->free_handles.end(), freed.begin(), freed.end());
  }
  return GF_OK;
}

}  // extern "C"
