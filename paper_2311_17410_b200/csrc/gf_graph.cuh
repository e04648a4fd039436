// gf_graph.cuh -- device-resident block store (reference storage.py DynamicGraph).
//
// HBM layout:
//   node table  (SoA, indexed by node id)      head, tail, num_blocks, degree (int64), node_valid (u8),
//                                              nslots (list end position), dir_off / dir_cap (block directory)
//   block arena (SoA, indexed by block handle) capacity, size, tmin, tmax, prev, next (int64, FastTier
//                                              columns storage.py:147-152) + base (slot-pool offset)
//   block directory (per node, contiguous)     32-byte entries {tmin, cum (list position of the first
//                                              slot), base, tmax}, one per block, head..tail, so the
//                                              sampler can search blocks instead of chasing prev pointers
//   slot pool  (AoS, 32 B per slot)            Slot{ts, eid, nbr, owner, valid}; block h owns
//                                              [base[h], base[h] + capacity[h])
//   sts        (int64 per slot)                dense copy of the slot timestamps (window reads)
//   fts        (int64 per 32 slots)            fence index: fts[i] = ts of pool slot 32*i, a sorted
//                                              subsequence of every block's timestamps (L2-sized)
//   sts32      (int32 per slot)                32-bit copy of the slot timestamps, exact while every
//                                              timestamp fits int32 (ts32): 32 per 128 B line
//   fts32      (int32 per 32 slots)            32-bit fence, fts32[i] = ts of pool slot 32*i (ts32):
//                                              29 MB at GDELT scale, and the 32-slot window it leaves
//                                              is ONE aligned line of sts32
//   nflags     (u8 per node)                   bit 0: block list not on the sizing law's closed form
//   okbits     (1 bit per slot, after the      slot is a candidate: valid edge and valid neighbour
//               first deletion)                (23 MB at GDELT scale: the post-deletion sampler's
//                                              validity checks stay in L2)
#pragma once

#include <atomic>
#include <vector>

#include "gf_common.cuh"

struct gf_graph {
  int device = 0;
  int directed = 0;
  int64_t tau = 48;
  int sizing_kind = GF_SIZING_ADAPTIVE;
  int64_t sizing_param = 0;

  int64_t num_nodes = 0, node_cap = 0;
  int64_t blk_used = 0, blk_cap = 0;
  int64_t slots_used = 0, slot_cap = 0;
  int64_t dir_used = 0, dir_cap_total = 0;
  int64_t next_edge_id = 0, total_edges_inserted = 0;
  std::vector<int64_t> free_handles;  // FastTier._free_handles (storage.py:154, 190-191)
  int any_deleted = 0;

  // node table
  int64_t *head = nullptr, *tail = nullptr, *num_blocks = nullptr, *degree = nullptr;
  uint8_t* node_valid = nullptr;
  int64_t *nslots = nullptr, *dir_off = nullptr, *dir_cap = nullptr;
  uint8_t* nflags = nullptr;
  int64_t* nrec = nullptr;  // packed 64-byte sampler record per node (NodeRec)
  // block arena
  int64_t *bcap = nullptr, *bsize = nullptr, *btmin = nullptr, *btmax = nullptr, *bprev = nullptr,
          *bnext = nullptr, *bbase = nullptr;
  // block directory pool
  int64_t* dir = nullptr;  // DIRW words per entry: tmin, cum, base, tmax
  // slot pool
  gf::Slot* slots = nullptr;
  int64_t* sts = nullptr;
  int64_t* fts = nullptr;
  int32_t* sts32 = nullptr;  // 32-bit slot timestamps (valid while ts32)
  int32_t* fts32 = nullptr;  // 32-bit fence every 32 slots (valid while ts32)
  int ts32 = 1;              // every timestamp ingested so far fits in int32
  // candidate bitmap, one bit per pool slot: valid edge and valid neighbour (sampling.py:178).
  // Allocated by the first deletion, rebuilt by every delete call, kept current by ingest.
  uint32_t* okbits = nullptr;
  // persistent ingest scratch (sync-free path), sized for the largest batch seen
  void* ing_buf = nullptr;
  size_t ing_bytes = 0;
  // ingest launch sequence captured as a CUDA graph, replayed while its key holds
  int64_t gen = 0;            // bumped whenever a pool or table is reallocated
  void* ing_host = nullptr;   // pinned: per-call scalars (H2D) + counters (D2H)
  cudaGraphExec_t ing_exec = nullptr;
  cudaStream_t cap_stream = nullptr;
  int64_t* free_dev = nullptr;  // device copy of free_handles for the commit kernel
  int64_t free_dev_cap = 0;
  int64_t ing_key[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  int64_t ing_nodes = 0;      // kernel launches per replay
  // cooperative single-launch ingest (gf_graph.cu k_ingest_coop): its own scratch, and two
  // per-node int32 arrays -- event counters (all zero between batches) and segment indices
  void* co_buf = nullptr;
  size_t co_bytes = 0;
  int32_t* co_ncnt = nullptr;
  int32_t* co_nseg = nullptr;
  int64_t co_node_cap = 0;
  // persistent sampling scratch (totals, per-hop tile state, child keys) + pinned totals; a call
  // that finds it busy (another stream) allocates its own
  void* smp_buf = nullptr;
  size_t smp_bytes = 0;
  int64_t* smp_host = nullptr;
  std::atomic<int> smp_busy{0};
};

namespace gf {

constexpr int FENCE = 32;    // pool slots per fence entry (int64 fence, general path)
constexpr int FENCE32 = 32;  // pool slots per 32-bit fence entry: a 32-slot window of sts32 is one 128 B line

// NodeRec: one 128-byte line per node, everything a sampler query needs first
// (one coalesced load): word 0 dir_off, 1 nslots (list end), 2 num_blocks |
// valid << 32 | irregular << 33, 3 first live list position, 4 tail block
// cum, 5 tail block slot base, 6 tail block tmin, 7 latest timestamp,
// 8 head block tmin, 9-15 reserved.
constexpr int NREC = 16;
constexpr int DIRW = 4;  // directory entry: tmin, cum, base, tmax
constexpr int64_t NREC_VALID = 1ll << 32;
constexpr int64_t NREC_IRREG = 1ll << 33;

// Closed-form block index of a list position for nodes whose blocks follow
// the sizing law exactly (no deletion before an allocation, no offload):
// adaptive caps are min(max(cum_b, 1), tau) (storage.py:88-89, degree ==
// slots written), so cum_b = 2^(b-1) up to the first b = m with
// 2^(b-1) >= tau, then grows by tau; fixed caps give cum_b = b * size.
struct SizingLaw {
  int kind;
  int64_t tau, size, m, cum_m;
  int tau_shift, size_shift;  // log2 when a power of two, else -1 (avoids 64-bit division)
};

inline int log2_exact(int64_t x) {
  if (x <= 0 || (x & (x - 1))) return -1;
  int s = 0;
  while ((1ll << s) < x) s++;
  return s;
}

inline SizingLaw sizing_law(int kind, int64_t tau, int64_t param) {
  SizingLaw L{kind, tau, param, 0, 0, log2_exact(tau), log2_exact(param)};
  if (kind == GF_SIZING_ADAPTIVE) {
    int64_t b = 1;
    while ((1ll << (b - 1)) < tau) b++;
    L.m = b;
    L.cum_m = 1ll << (b - 1);
  }
  return L;
}

// read-only view passed to sampling kernels
struct GraphView {
  const uint8_t* node_valid;
  const int64_t* num_blocks;
  const int64_t* nslots;
  const int64_t* dir_off;
  const int64_t* dir;
  const Slot* slots;
  const int64_t* sts;
  const int64_t* fts;
  const int32_t* sts32;
  const int32_t* fts32;
  const uint8_t* nflags;
  const int64_t* nrec;
  const uint32_t* okbits;  // NULL until the first deletion
  int64_t num_nodes;
  int any_deleted;
  int ts32;
  SizingLaw law;
};

inline GraphView view_of(const gf_graph* g) {
  return GraphView{g->node_valid, g->num_blocks, g->nslots, g->dir_off,   g->dir,
                   g->slots,      g->sts,        g->fts,       g->sts32,     g->fts32,     g->nflags,
                   g->nrec,       g->okbits,    g->num_nodes,  g->any_deleted, g->ts32,
                   sizing_law(g->sizing_kind, g->tau, g->sizing_param)};
}

}  // namespace gf
