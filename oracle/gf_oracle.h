/*
 * gf_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's block store and temporal sampler
 * (/root/reference/pkg/src/ctdg/storage.py, sampling.py).  It exists to CHECK
 * the CUDA path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_2311_17410_b200/libgfb200.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here
 * against fixtures produced by the unmodified reference
 * (tests/golden/make_golden.py).  The one deliberate deviation from the
 * reference is the uniform/time-window RNG stream: the reference draws with
 * numpy PCG64 seeded per (seed, node, window, occurrence)
 * (sampling.py:140-142,191-198); this oracle uses the Philox4x32-10 + Floyd
 * scheme the GPU uses, so GPU uniform output
 * can be compared bit-for-bit with the oracle, while the reference's
 * distribution is checked statistically.
 */
#ifndef GF_ORACLE_H
#define GF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_graph or_graph;

/* sizing kinds mirror storage.py:74-121 */
#define OR_SIZING_ADAPTIVE 0
#define OR_SIZING_FIXED 1
#define OR_SIZING_BATCH 2

/* policy codes mirror wire.py:27 / sampling.py:28 */
#define OR_RECENT 0
#define OR_UNIFORM 1
#define OR_TIME_WINDOW 2

or_graph* or_graph_create(int directed, int64_t tau, int sizing_kind, int64_t sizing_param);
void or_graph_destroy(or_graph* g);

/* storage.py:394-450.  out_eids[i] = assigned id or -1 when rejected.
 * Returns number of rejected edges, or -1 for a negative node id (ValueError). */
int64_t or_add_edges(or_graph* g, const int64_t* src, const int64_t* dst, const int64_t* ts,
                     int64_t n, const int64_t* eids_in, int64_t* out_eids);
/* storage.py:479-505: returns number of ids actually deleted */
int64_t or_delete_edges(or_graph* g, const int64_t* eids, int64_t n);
/* storage.py:507-512 */
int or_delete_node(or_graph* g, int64_t node);

/* storage.py:516-574: writes the TGOF blob and unlinks; -1 if cap too small */
int64_t or_offload_before(or_graph* g, int64_t cutoff, uint8_t* blob, int64_t cap, int64_t* blob_len);
int64_t or_num_nodes(const or_graph* g);
int64_t or_num_block_handles(const or_graph* g);
int64_t or_next_edge_id(const or_graph* g);
int64_t or_total_edges_inserted(const or_graph* g);
/* FastTier columns (storage.py:140-152) copied out */
void or_export_nodes(const or_graph* g, int64_t* head, int64_t* tail, int64_t* num_blocks,
                     int64_t* degree, uint8_t* node_valid);
void or_export_blocks(const or_graph* g, int64_t* cap, int64_t* size, int64_t* tmin, int64_t* tmax,
                      int64_t* prev, int64_t* next);
/* SharedTier arrays of one block, first `size` slots (storage.py:201-238) */
int64_t or_export_block_edges(const or_graph* g, int64_t handle, int64_t* nbr, int64_t* eid,
                              int64_t* ts, uint8_t* valid);

/* sampling.py:219-273 (+ _collect_candidates :145-182, _select :185-198).
 * keys: per-query RNG key (NULL => query index).  Writes at most out_cap
 * edges; always returns the total number of sampled edges.  offsets has n+1
 * entries.  threads: worker threads (output is thread-count invariant).
 * faithful=1 collects every in-window candidate the way the reference does
 * (O(candidates) per query); faithful=0 stops early (same output).
 * Returns -1 on invalid arguments. */
int64_t or_sample_layer(const or_graph* g, const int64_t* src, const int64_t* t_start,
                        const int64_t* t_end, int64_t n, int64_t fanout, int policy, int64_t delta,
                        uint64_t seed, const uint64_t* keys, int64_t* offsets, int64_t* out_nbr,
                        int64_t* out_eid, int64_t* out_ts, int64_t out_cap, int threads,
                        int faithful);

/* Multi-hop driver (sampling.py:276-299) with path-derived query keys.
 * fanouts[n_hops]; per-hop outputs are caller arrays; caps per hop.
 * totals[h] receives each hop's total; returns 0, or -1 on bad args,
 * or -2 if some hop's output exceeded its cap (totals still filled up to it). */
int or_sample_khop(const or_graph* g, const int64_t* roots, const int64_t* ts, int64_t n_roots,
                   const int64_t* fanouts, int n_hops, int policy, int64_t delta, uint64_t seed,
                   uint64_t root_key_base, int64_t** offsets, int64_t** out_nbr,
                   int64_t** out_eid, int64_t** out_ts, const int64_t* caps, int64_t* totals,
                   int threads, int faithful);

/* sampling.py:135-137: SeedSequence([seed, hop]).generate_state(1, uint64)[0] */
uint64_t or_hop_seed(uint64_t seed, uint64_t hop);
/* child query key */
uint64_t or_child_key(uint64_t parent, uint64_t j);
/* Philox4x32-10 (Salmon et al. 2011), exposed for tests */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif
#endif
