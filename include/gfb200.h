/*
 * gfb200.h -- C ABI of the B200-native GNNFlow hot path (libgfb200.so).
 *
 * Drop-in boundary for the reference's Python API (package `ctdg`,
 * /root/reference/pkg/src/ctdg).  The reference has no FFI of its own; each
 * entry point below replaces one reference call, cited as file:line
 * (relative to /root/reference/pkg/src/ctdg/).  INTEGRATION.md shows the
 * ctypes binding a reference maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Arrays named d_* are DEVICE pointers
 *    (CUDA global memory on the handle's device); h_* are HOST pointers.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All work is stream-ordered; functions that must return a host value
 *    (counts, status of data-dependent validation) synchronise the stream.
 *  - Every function returns a gf_status.  On error, gf_last_error() returns a
 *    thread-local message.  The Python facade maps GF_EINVAL -> ValueError,
 *    GF_ENOTFOUND -> NodeNotFoundError (KeyError), GF_ERANGE -> "output
 *    buffer too small, retry with *out_total".
 *  - ids and timestamps are int64 exactly as in the reference; node ids must
 *    be < 2^31 (the node table is dense up to the largest id, storage.py:406-412).
 *  - A handle is not safe for concurrent mutation; concurrent read-only
 *    sampling on different streams is safe.
 */
#ifndef GFB200_H
#define GFB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  GF_OK = 0,
  GF_EINVAL = 1,     /* ValueError in the reference */
  GF_ENOTFOUND = 2,  /* NodeNotFoundError (storage.py:53-54) */
  GF_ENOMEM = 3,
  GF_ECUDA = 4,
  GF_ERANGE = 5,     /* caller output buffer too small; *out_total holds the need */
  GF_EFORMAT = 6     /* malformed snapshot / state */
} gf_status;

/* sizing kinds: storage.py:74-121 */
enum { GF_SIZING_ADAPTIVE = 0, GF_SIZING_FIXED = 1, GF_SIZING_BATCH = 2 };
/* sampling policy codes: wire.py:27, sampling.py:28 */
enum { GF_POLICY_RECENT = 0, GF_POLICY_UNIFORM = 1, GF_POLICY_TIME_WINDOW = 2 };
/* cache policy codes: cache.py:27 */
enum { GF_CACHE_LRU = 0, GF_CACHE_LFU = 1, GF_CACHE_FIFO = 2 };

typedef struct gf_graph gf_graph;
typedef struct gf_cache gf_cache;
typedef struct gf_cache_snap gf_cache_snap;
typedef struct gf_ftable gf_ftable;

const char* gf_last_error(void);
/* library version string */
const char* gf_version(void);
/* number of kernels this process has launched through the library */
uint64_t gf_launch_count(void);
/* Per-kernel CUDA-event timing of every library launch (off by default;
 * enabling clears previous records).  gf_profile_summary writes one line per
 * kernel: "name<TAB>launches<TAB>total_ms" (synchronises the device). */
void gf_profile_enable(int on);
gf_status gf_profile_summary(char* buf, int64_t len);

/* ---- hop seeds -------------------------------------------------------- */
/* sampling.py:135-137 hop_seed(seed, hop) = SeedSequence([seed, hop]).generate_state(1, u64)[0] */
uint64_t gf_hop_seed(uint64_t seed, uint64_t hop);
/* key of the j-th sampled edge of a query with key `parent` */
uint64_t gf_child_key(uint64_t parent, uint64_t j);

/* ---- block store: storage.py DynamicGraph ------------------------------ */
/* DynamicGraph.__init__ / new_graph (storage.py:312-323, 620-621).
 * tau < 1 with adaptive sizing, or fixed size < 1 -> GF_EINVAL. */
gf_status gf_graph_create(int directed, int64_t tau, int sizing_kind, int64_t sizing_param, int device,
                          gf_graph** out);
gf_status gf_graph_destroy(gf_graph* g);
/* Pre-size device arrays (optional; they also grow geometrically). */
gf_status gf_graph_reserve(gf_graph* g, int64_t nodes, int64_t blocks, int64_t slots, void* stream);

/* DynamicGraph.add_edges (storage.py:394-450) + _append_edge (:452-477).
 * d_src/d_dst/d_ts: n edges in arrival order.  d_eids_in: preassigned ids or
 * NULL.  d_out_eids[i] = assigned id, or -1 for an edge rejected as out of
 * order (ts < latest ts at a stored endpoint).  *h_out_rejected = number of
 * rejected edges.  Negative node id -> GF_EINVAL (nothing applied). */
gf_status gf_graph_add_edges(gf_graph* g, const int64_t* d_src, const int64_t* d_dst, const int64_t* d_ts,
                             int64_t n, const int64_t* d_eids_in, int64_t* d_out_eids, int64_t* h_out_rejected,
                             void* stream);
/* DynamicGraph.delete_edges (storage.py:479-505): *h_out_deleted = distinct live ids deleted */
gf_status gf_graph_delete_edges(gf_graph* g, const int64_t* d_eids, int64_t n, int64_t* h_out_deleted,
                                void* stream);
/* DynamicGraph.delete_node (storage.py:507-512): *h_out_deleted = 1 if the node was live */
gf_status gf_graph_delete_node(gf_graph* g, int64_t node, int* h_out_deleted, void* stream);

/* DynamicGraph.offload_before (storage.py:516-574): blocks with tmax < cutoff
 * that form a prefix of their node's list are serialised to a TGOF blob
 * (storage.py:535-556) and, if `commit`, unlinked (head/tail/num_blocks/live
 * degree; freed handles are reused LIFO by later appends, storage.py:171-191).
 * *h_blob_len = blob size; *h_edges = edge records in it.  h_blob (host, may be
 * NULL) receives the blob when blob_cap is large enough (else GF_ERANGE).
 * Call with commit = 0 to fetch the blob, write it, then commit = 1: the
 * graph is unchanged until the commit call. */
gf_status gf_graph_offload_before(gf_graph* g, int64_t cutoff, uint8_t* h_blob, int64_t blob_cap, int64_t* h_blob_len,
                                  int64_t* h_edges, int commit, void* stream);

typedef struct {
  int64_t num_nodes;            /* storage.py:327-329 */
  int64_t num_block_handles;    /* arena length (FastTier._blk_used) */
  int64_t live_blocks;          /* FastTier.live_blocks */
  int64_t slots_allocated;      /* sum of live block capacities */
  int64_t next_edge_id;         /* storage.py:322 */
  int64_t total_edges_inserted; /* storage.py:323 */
  int64_t any_deleted;          /* 1 once any edge/node deletion succeeded */
  int64_t directed, tau, sizing_kind, sizing_param;
  int64_t device_bytes;         /* device memory held by the handle */
} gf_graph_info;
gf_status gf_graph_get_info(gf_graph* g, gf_graph_info* out);

/* Host mirrors of FastTier columns (storage.py:140-152) for parity checks.
 * Node arrays have info.num_nodes entries, block arrays info.num_block_handles.
 * Any pointer may be NULL.  Synchronous. */
gf_status gf_graph_export_nodes(gf_graph* g, int64_t* h_head, int64_t* h_tail, int64_t* h_num_blocks,
                                int64_t* h_degree, uint8_t* h_node_valid, void* stream);
gf_status gf_graph_export_blocks(gf_graph* g, int64_t* h_capacity, int64_t* h_size, int64_t* h_tmin,
                                 int64_t* h_tmax, int64_t* h_prev, int64_t* h_next, void* stream);
/* SharedTier edge arrays (storage.py:201-238) of blocks [h0, h1): slots of
 * block h occupy [h_offsets[h-h0], h_offsets[h-h0+1]) of the outputs
 * (h_offsets has h1-h0+1 entries; only `size` slots are exported). */
gf_status gf_graph_export_slots(gf_graph* g, int64_t h0, int64_t h1, int64_t* h_offsets, int64_t* h_nbr,
                                int64_t* h_eid, int64_t* h_ts, uint8_t* h_valid, void* stream);

/* ---- temporal sampler: sampling.py ------------------------------------ */
/* sample_layer (sampling.py:219-273) for n queries (d_src, d_t_start, d_t_end).
 * d_t_start may be NULL (= TS_MIN for every query, as sample_khop passes).
 * policy: GF_POLICY_*; delta > 0 required for time_window.
 * seed: the hop's RNG key (sample_khop passes gf_hop_seed(seed, hop)).
 * d_keys: per-query RNG keys or NULL (= query index + key_base).
 * Outputs: d_offsets[n+1], and d_nbr/d_eid/d_ts with capacity out_cap.
 * *h_out_total = number of sampled edges; GF_ERANGE if it exceeds out_cap
 * (nothing written beyond offsets).  d_out_keys (optional, capacity out_cap)
 * receives each sampled edge's child key for chaining another hop. */
gf_status gf_sample_layer(gf_graph* g, const int64_t* d_src, const int64_t* d_t_start, const int64_t* d_t_end,
                          int64_t n, int64_t fanout, int policy, int64_t delta, uint64_t seed,
                          const uint64_t* d_keys, uint64_t key_base, int64_t* d_offsets, int64_t* d_nbr,
                          int64_t* d_eid, int64_t* d_ts, uint64_t* d_out_keys, int64_t out_cap,
                          int64_t* h_out_total, void* stream);

/* sample_khop (sampling.py:276-299): hop 0 queries (d_roots, TS_MIN, d_ts);
 * hop l+1 queries (hop-l neighbors, TS_MIN, hop-l timestamps).  Per-hop
 * outputs are caller buffers: d_offsets[h] (length n_h+1, n_0 = n_roots,
 * n_{h+1} = total_h), d_nbr[h], d_eid[h], d_ts[h] with capacity caps[h].
 * RNG: hop h uses gf_hop_seed(seed, h); root i has key root_key_base + i, so
 * a root batch split across ranks with matching bases reproduces the
 * single-GPU sample bit-for-bit.  h_totals[h] = per-hop totals.  GF_ERANGE
 * when a hop overflows its cap (h_totals filled up to that hop). */
gf_status gf_sample_khop(gf_graph* g, const int64_t* d_roots, const int64_t* d_ts, int64_t n_roots,
                         const int64_t* h_fanouts, int n_hops, int policy, int64_t delta, uint64_t seed,
                         uint64_t root_key_base, int64_t* const* d_offsets, int64_t* const* d_nbr,
                         int64_t* const* d_eid, int64_t* const* d_ts_out, const int64_t* h_caps, int64_t* h_totals,
                         void* stream);

/* ---- vectorised feature cache: cache.py VectorCache -------------------- */
/* VectorCache.__init__ (cache.py:56-74); bad policy/capacity/lam -> GF_EINVAL */
gf_status gf_cache_create(int policy, int64_t capacity, int64_t dim, double lam, int device, gf_cache** out);
gf_status gf_cache_destroy(gf_cache* c);
/* VectorCache.fetch (cache.py:85-121).  d_values [n x dim] fp32 row-major
 * (zeros for misses), d_hit[n] (0/1), d_miss_keys (capacity n) receives the
 * missed keys deduplicated in first-occurrence order; *h_n_miss their count
 * (synchronous). */
gf_status gf_cache_fetch(gf_cache* c, const int64_t* d_keys, int64_t n, float* d_values, uint8_t* d_hit,
                         int64_t* d_miss_keys, int64_t* h_n_miss, void* stream);
/* VectorCache.insert_batch (cache.py:123-177).  d_values [n x dim].
 * A key already cached -> GF_EINVAL (nothing applied).  *h_admitted = number
 * of entries admitted (<= floor(lam * capacity)). */
gf_status gf_cache_insert(gf_cache* c, const int64_t* d_keys, int64_t n, const float* d_values,
                          int64_t* h_admitted, void* stream);
/* VectorCache.stats / reset_stats (cache.py:223-233) */
gf_status gf_cache_stats(gf_cache* c, int64_t* h_hits, int64_t* h_misses, int64_t* h_evictions);
gf_status gf_cache_reset_stats(gf_cache* c);
/* Raw state access (keys/scores int64[capacity], storage fp32[capacity x dim],
 * fifo_head) for snapshot files (cache.py:205-273) and parity checks.
 * set_state rebuilds the key->slot map (cache.py:193-203). Synchronous. */
gf_status gf_cache_get_state(gf_cache* c, int64_t* h_keys, int64_t* h_scores, float* h_storage,
                             int64_t* h_fifo_head, void* stream);
gf_status gf_cache_set_state(gf_cache* c, const int64_t* h_keys, const int64_t* h_scores, const float* h_storage,
                             int64_t fifo_head, void* stream);
/* Device-resident snapshot / restore (cache.py:181-203), for per-epoch restoration */
gf_status gf_cache_snapshot(gf_cache* c, gf_cache_snap** out, void* stream);
gf_status gf_cache_restore(gf_cache* c, const gf_cache_snap* s, void* stream);
gf_status gf_cache_snapshot_free(gf_cache_snap* s);

/* ---- feature tables: features.py --------------------------------------- */
/* kind 0 = NodeFeatureTable (features.py:27-61; upsert by id, dense id index),
 * kind 1 = EdgeFeatureTable (features.py:64-120; append strictly increasing ids,
 * binary-search lookup). */
gf_status gf_ftable_create(int kind, int64_t dim, int device, gf_ftable** out);
gf_status gf_ftable_destroy(gf_ftable* t);
/* node: set rows for ids (last write wins); edge: append (ids strictly
 * increasing and above the current max, else GF_EINVAL) */
gf_status gf_ftable_put(gf_ftable* t, const int64_t* d_ids, int64_t n, const float* d_rows, void* stream);
/* NodeFeatureTable.get / EdgeFeatureTable.get: rows (zeros if unknown) + found mask */
gf_status gf_ftable_get(gf_ftable* t, const int64_t* d_ids, int64_t n, float* d_rows, uint8_t* d_found,
                        void* stream);
gf_status gf_ftable_size(gf_ftable* t, int64_t* h_n);
/* Stored ids in ascending order (NodeFeatureTable.ids_sorted, features.py:60-61;
 * EdgeFeatureTable.ids, features.py:76-78) into d_ids[cap]; *h_n = the count.
 * GF_ERANGE (with *h_n set) when cap is too small.  Used by save_*_features. */
gf_status gf_ftable_ids(gf_ftable* t, int64_t* d_ids, int64_t cap, int64_t* h_n, void* stream);

/* Harness fetch block (harness.py:438-446): cache.fetch(keys) -> table.get(miss)
 * -> cache.insert_batch(found rows), one call.  d_values [n x dim] receives the
 * COMPLETE row of every key: the cached row for a hit, the table row for a miss
 * whose id the table holds, zeros for an id the table does not hold (the
 * reference harness discards fetch's values, harness.py:438,443, so the block
 * returns the rows a trainer would consume).  d_hit[n] is the cache hit mask.
 * *h_n_miss = distinct missed keys, *h_admitted = rows the insert admitted.
 * Returns with the insert still queued on `stream`: readers of the cache state
 * on other streams synchronise (gf_cache_stats / get_state / snapshot do). */
gf_status gf_fetch_features(gf_cache* c, gf_ftable* t, const int64_t* d_keys, int64_t n, float* d_values,
                            uint8_t* d_hit, int64_t* h_n_miss, int64_t* h_admitted, void* stream);

/* Row gather (K6): out[i, :] = table[idx[i], :] (ld = row pitch in floats);
 * idx < 0 -> zero row. */
gf_status gf_gather_rows(const float* d_table, int64_t ld, const int64_t* d_idx, int64_t n, int64_t dim,
                         float* d_out, void* stream);

/* ---- multi-GPU exchange helpers (gf_part.cu) ---------- */
/* Stable bucketing by owner = key mod nparts (floor modulo, partition.py:38-39; cluster.py:244
 * routes queries by src % machines, cluster.py:296-325 feature ids by owner).  d_perm[j] = index
 * of the j-th key in send order (owner-major, original order inside an owner); d_keys_out (may be
 * NULL) = keys in that order; h_counts[p] = keys owned by p (host, synchronous).  1 <= nparts <= 64. */
gf_status gf_bucket_by_owner(const int64_t* d_keys, int64_t n, int nparts, int64_t* d_perm, int64_t* d_keys_out,
                             int64_t* h_counts, void* stream);
/* Merge owner answers back into request order (cluster.py:268-292): query j of the send order
 * (d_perm[j] = its original index) returned d_cnt_sorted[j] edges, stored consecutively in each
 * of the narr (<= 8) arrays d_in[a] (send order).  Writes d_offsets[n+1] (original order, CSR)
 * and d_out[a] (original order); *h_total = edges (synchronous). */
gf_status gf_csr_merge(const int64_t* d_perm, const int64_t* d_cnt_sorted, int64_t n, int narr,
                       const int64_t* const* d_in, int64_t* d_offsets, int64_t* const* d_out, int64_t* h_total,
                       void* stream);
/* Row scatter: out[dest[i], :] = in[i, :] (row pitches ld_in / ld_out in floats) -- feature rows
 * answered by their owners back into request order. */
gf_status gf_scatter_rows(const float* d_in, int64_t ld_in, const int64_t* d_dest, int64_t n, int64_t dim, float* d_out,
                          int64_t ld_out, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* GFB200_H */
