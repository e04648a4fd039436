/*
 * gf_oracle.c -- CPU ORACLE (test infrastructure only; see gf_oracle.h).
 *
 * Plain-C restatement of the reference block store + temporal sampler.
 * Every function cites the reference lines it follows
 * (paths relative to /root/reference/pkg/src/ctdg/).
 * Never linked into, or called from, the product path.
 */
#include "gf_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define NO_BLOCK (-1)                      /* storage.py:31 */
#define TS_MIN ((int64_t)(-9223372036854775807LL - 1)) /* storage.py:45 */

typedef struct {
  int64_t* nbr; /* SharedTier/EdgeArrays, storage.py:201-217 */
  int64_t* eid;
  int64_t* ts;
  uint8_t* valid;
} or_edges;

struct or_graph {
  int directed;
  int64_t tau;
  int sizing_kind;
  int64_t sizing_param;
  /* FastTier node columns, storage.py:140-145 */
  int64_t n_nodes, node_alloc;
  int64_t *head, *tail, *num_blocks, *degree;
  uint8_t* node_valid;
  /* FastTier block columns, storage.py:147-154 */
  int64_t blk_used, blk_alloc;
  int64_t *cap, *size, *tmin, *tmax, *prev, *next;
  or_edges* edges;
  int64_t *free_handles, n_free, free_alloc;
  int64_t next_edge_id, total_edges_inserted; /* storage.py:322-323 */
};

static void* xrealloc(void* p, size_t n) {
  void* q = realloc(p, n ? n : 1);
  if (!q) abort();
  return q;
}

or_graph* or_graph_create(int directed, int64_t tau, int sizing_kind, int64_t sizing_param) {
  /* storage.py:312-323 (tau < 1 -> ValueError is checked by the caller) */
  or_graph* g = (or_graph*)calloc(1, sizeof(or_graph));
  g->directed = directed;
  g->tau = tau;
  g->sizing_kind = sizing_kind;
  g->sizing_param = sizing_param;
  return g;
}

void or_graph_destroy(or_graph* g) {
  if (!g) return;
  for (int64_t h = 0; h < g->blk_used; h++) {
    free(g->edges[h].nbr);
    free(g->edges[h].eid);
    free(g->edges[h].ts);
    free(g->edges[h].valid);
  }
  free(g->edges);
  free(g->head); free(g->tail); free(g->num_blocks); free(g->degree); free(g->node_valid);
  free(g->cap); free(g->size); free(g->tmin); free(g->tmax); free(g->prev); free(g->next);
  free(g->free_handles);
  free(g);
}

/* FastTier.grow_nodes, storage.py:160-169 */
static void grow_nodes(or_graph* g, int64_t new_size) {
  if (new_size <= g->n_nodes) return;
  if (new_size > g->node_alloc) {
    int64_t a = g->node_alloc ? g->node_alloc : 16;
    while (a < new_size) a *= 2;
    g->head = xrealloc(g->head, a * 8);
    g->tail = xrealloc(g->tail, a * 8);
    g->num_blocks = xrealloc(g->num_blocks, a * 8);
    g->degree = xrealloc(g->degree, a * 8);
    g->node_valid = xrealloc(g->node_valid, a);
    g->node_alloc = a;
  }
  for (int64_t v = g->n_nodes; v < new_size; v++) {
    g->head[v] = NO_BLOCK;
    g->tail[v] = NO_BLOCK;
    g->num_blocks[v] = 0;
    g->degree[v] = 0;
    g->node_valid[v] = 1;
  }
  g->n_nodes = new_size;
}

/* FastTier.alloc_block + SharedTier.alloc, storage.py:171-188, 227-230 */
static int64_t alloc_block(or_graph* g, int64_t capacity) {
  int64_t h;
  if (g->n_free) {
    h = g->free_handles[--g->n_free]; /* list.pop(): LIFO */
  } else {
    if (g->blk_used == g->blk_alloc) {
      int64_t grow = g->blk_alloc > 64 ? g->blk_alloc : 64;
      int64_t a = g->blk_alloc + grow;
      g->cap = xrealloc(g->cap, a * 8);
      g->size = xrealloc(g->size, a * 8);
      g->tmin = xrealloc(g->tmin, a * 8);
      g->tmax = xrealloc(g->tmax, a * 8);
      g->prev = xrealloc(g->prev, a * 8);
      g->next = xrealloc(g->next, a * 8);
      g->edges = xrealloc(g->edges, a * sizeof(or_edges));
      memset(g->edges + g->blk_alloc, 0, (a - g->blk_alloc) * sizeof(or_edges));
      g->blk_alloc = a;
    }
    h = g->blk_used++;
  }
  g->cap[h] = capacity;
  g->size[h] = 0;
  g->tmin[h] = 0;
  g->tmax[h] = 0;
  g->prev[h] = NO_BLOCK;
  g->next[h] = NO_BLOCK;
  or_edges* e = &g->edges[h];
  free(e->nbr); free(e->eid); free(e->ts); free(e->valid);
  e->nbr = (int64_t*)calloc(capacity, 8);
  e->eid = (int64_t*)calloc(capacity, 8);
  e->ts = (int64_t*)calloc(capacity, 8);
  e->valid = (uint8_t*)calloc(capacity, 1);
  return h;
}

/* BlockSizing.capacity, storage.py:88-89, 102-103, 116-117 */
static int64_t sizing_capacity(const or_graph* g, int64_t degree, int64_t pending) {
  switch (g->sizing_kind) {
    case OR_SIZING_FIXED: return g->sizing_param;
    case OR_SIZING_BATCH: return pending > 1 ? pending : 1;
    default: {
      int64_t d = degree > 1 ? degree : 1;
      return d < g->tau ? d : g->tau;
    }
  }
}

/* DynamicGraph.node_t_max, storage.py:382-390 */
static int64_t node_t_max(const or_graph* g, int64_t v) {
  int64_t t = (v >= 0 && v < g->n_nodes) ? g->tail[v] : NO_BLOCK;
  if (t == NO_BLOCK) return TS_MIN;
  int64_t s = g->size[t];
  if (s == 0) return TS_MIN;
  return g->edges[t].ts[s - 1];
}

/* DynamicGraph._append_edge, storage.py:452-477 */
static void append_edge(or_graph* g, int64_t node, int64_t nbr, int64_t eid, int64_t ts,
                        int64_t pending) {
  int64_t tail = g->tail[node];
  if (tail == NO_BLOCK || g->size[tail] == g->cap[tail]) {
    int64_t cap = sizing_capacity(g, g->degree[node], pending);
    int64_t h = alloc_block(g, cap);
    if (tail == NO_BLOCK) {
      g->head[node] = h;
    } else {
      g->next[tail] = h;
      g->prev[h] = tail;
    }
    g->tail[node] = h;
    g->num_blocks[node] += 1;
    tail = h;
  }
  or_edges* e = &g->edges[tail];
  int64_t pos = g->size[tail];
  e->nbr[pos] = nbr;
  e->eid[pos] = eid;
  e->ts[pos] = ts;
  e->valid[pos] = 1;
  if (pos == 0) g->tmin[tail] = ts;
  g->tmax[tail] = ts;
  g->size[tail] = pos + 1;
  g->degree[node] += 1;
}

/* DynamicGraph.add_edges, storage.py:394-450 */
int64_t or_add_edges(or_graph* g, const int64_t* src, const int64_t* dst, const int64_t* ts,
                     int64_t n, const int64_t* eids_in, int64_t* out_eids) {
  int64_t max_node = -1;
  for (int64_t i = 0; i < n; i++) { /* :406-412 */
    if (src[i] < 0 || dst[i] < 0) return -1;
    if (src[i] > max_node) max_node = src[i];
    if (dst[i] > max_node) max_node = dst[i];
  }
  if (max_node >= g->n_nodes) grow_nodes(g, max_node + 1);
  /* pending counts, :417-421 */
  int64_t* pending = (int64_t*)calloc(g->n_nodes ? g->n_nodes : 1, 8);
  for (int64_t i = 0; i < n; i++) {
    pending[src[i]]++;
    if (!g->directed) pending[dst[i]]++;
  }
  int64_t rejected = 0;
  for (int64_t i = 0; i < n; i++) { /* :426-449 */
    int64_t s = src[i], d = dst[i], t = ts[i];
    int ok = t >= node_t_max(g, s);
    if (!g->directed && t < node_t_max(g, d)) ok = 0;
    if (!ok) {
      rejected++;
      out_eids[i] = -1;
      pending[s]--;
      if (!g->directed) pending[d]--;
      continue;
    }
    int64_t eid;
    if (eids_in) {
      eid = eids_in[i];
      if (eid + 1 > g->next_edge_id) g->next_edge_id = eid + 1;
    } else {
      eid = g->next_edge_id++;
    }
    append_edge(g, s, d, eid, t, pending[s]);
    pending[s]--;
    if (!g->directed) {
      append_edge(g, d, s, eid, t, pending[d]);
      pending[d]--;
    }
    out_eids[i] = eid;
    g->total_edges_inserted++;
  }
  free(pending);
  return rejected;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* DynamicGraph.delete_edges_set, storage.py:487-505 */
int64_t or_delete_edges(or_graph* g, const int64_t* eids, int64_t n) {
  if (n <= 0) return 0;
  int64_t* w = (int64_t*)malloc(n * 8);
  memcpy(w, eids, n * 8);
  qsort(w, n, 8, cmp_i64);
  /* count distinct ids actually deleted (a set in the reference) */
  uint8_t* hit = (uint8_t*)calloc(n, 1);
  for (int64_t v = 0; v < g->n_nodes; v++) {
    for (int64_t h = g->head[v]; h != NO_BLOCK; h = g->next[h]) {
      or_edges* e = &g->edges[h];
      for (int64_t i = 0; i < g->size[h]; i++) {
        int64_t* p = (int64_t*)bsearch(&e->eid[i], w, n, 8, cmp_i64);
        if (p && e->valid[i]) {
          e->valid[i] = 0;
          g->degree[v] -= 1;
          while (p > w && p[-1] == *p) p--;
          hit[p - w] = 1;
        }
      }
    }
  }
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; i++) cnt += hit[i];
  free(hit);
  free(w);
  return cnt;
}

/* DynamicGraph.delete_node, storage.py:507-512 */
int or_delete_node(or_graph* g, int64_t node) {
  if (node < 0 || node >= g->n_nodes || !g->node_valid[node]) return 0;
  g->node_valid[node] = 0;
  return 1;
}

static void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; i++) p[i] = (uint8_t)(v >> (8 * i));
}

/* DynamicGraph.offload_before, storage.py:516-574 (TGOF blob into `blob`).
 * Returns the number of edge records, or -1 when the blob does not fit
 * (nothing is unlinked then, as when the reference's sink.write fails). */
int64_t or_offload_before(or_graph* g, int64_t cutoff, uint8_t* blob, int64_t cap, int64_t* blob_len) {
  int64_t bytes = 8, n_edges = 0;
  for (int64_t v = 0; v < g->n_nodes; v++)
    for (int64_t h = g->head[v]; h != NO_BLOCK && g->tmax[h] < cutoff && g->size[h] > 0; h = g->next[h]) {
      bytes += 12 + 25 * g->size[h];
      n_edges += g->size[h];
    }
  *blob_len = bytes;
  if (!blob || cap < bytes) return -1;
  memcpy(blob, "TGOF", 4); /* :536-537 */
  put_le(blob + 4, 1, 4);
  uint8_t* p = blob + 8;
  for (int64_t v = 0; v < g->n_nodes; v++) /* :539-554 */
    for (int64_t h = g->head[v]; h != NO_BLOCK && g->tmax[h] < cutoff && g->size[h] > 0; h = g->next[h]) {
      put_le(p, (uint64_t)v, 8);
      put_le(p + 8, (uint64_t)g->size[h], 4);
      p += 12;
      for (int64_t i = 0; i < g->size[h]; i++) {
        put_le(p, (uint64_t)g->edges[h].nbr[i], 8);
        put_le(p + 8, (uint64_t)g->edges[h].eid[i], 8);
        put_le(p + 16, (uint64_t)g->edges[h].ts[i], 8);
        p[24] = g->edges[h].valid[i] ? 1 : 0;
        p += 25;
      }
    }
  for (int64_t v = 0; v < g->n_nodes; v++) { /* unlink, :558-573 */
    int64_t h = g->head[v], k = 0, live = 0;
    while (h != NO_BLOCK && g->tmax[h] < cutoff && g->size[h] > 0) {
      for (int64_t i = 0; i < g->size[h]; i++) live += g->edges[h].valid[i] != 0;
      if (g->n_free == g->free_alloc) {
        g->free_alloc = g->free_alloc ? 2 * g->free_alloc : 64;
        g->free_handles = xrealloc(g->free_handles, g->free_alloc * 8);
      }
      g->free_handles[g->n_free++] = h;
      k++;
      h = g->next[h];
    }
    if (!k) continue;
    g->head[v] = h;
    if (h == NO_BLOCK) g->tail[v] = NO_BLOCK;
    else g->prev[h] = NO_BLOCK;
    g->num_blocks[v] -= k;
    g->degree[v] -= live;
  }
  return n_edges;
}

int64_t or_num_nodes(const or_graph* g) { return g->n_nodes; }
int64_t or_num_block_handles(const or_graph* g) { return g->blk_used; }
int64_t or_next_edge_id(const or_graph* g) { return g->next_edge_id; }
int64_t or_total_edges_inserted(const or_graph* g) { return g->total_edges_inserted; }

void or_export_nodes(const or_graph* g, int64_t* head, int64_t* tail, int64_t* num_blocks,
                     int64_t* degree, uint8_t* node_valid) {
  int64_t n = g->n_nodes;
  if (head) memcpy(head, g->head, n * 8);
  if (tail) memcpy(tail, g->tail, n * 8);
  if (num_blocks) memcpy(num_blocks, g->num_blocks, n * 8);
  if (degree) memcpy(degree, g->degree, n * 8);
  if (node_valid) memcpy(node_valid, g->node_valid, n);
}

void or_export_blocks(const or_graph* g, int64_t* cap, int64_t* size, int64_t* tmin, int64_t* tmax,
                      int64_t* prev, int64_t* next) {
  int64_t n = g->blk_used;
  if (cap) memcpy(cap, g->cap, n * 8);
  if (size) memcpy(size, g->size, n * 8);
  if (tmin) memcpy(tmin, g->tmin, n * 8);
  if (tmax) memcpy(tmax, g->tmax, n * 8);
  if (prev) memcpy(prev, g->prev, n * 8);
  if (next) memcpy(next, g->next, n * 8);
}

int64_t or_export_block_edges(const or_graph* g, int64_t h, int64_t* nbr, int64_t* eid,
                              int64_t* ts, uint8_t* valid) {
  if (h < 0 || h >= g->blk_used) return -1;
  int64_t s = g->size[h];
  const or_edges* e = &g->edges[h];
  if (nbr) memcpy(nbr, e->nbr, s * 8);
  if (eid) memcpy(eid, e->eid, s * 8);
  if (ts) memcpy(ts, e->ts, s * 8);
  if (valid) memcpy(valid, e->valid, s);
  return s;
}

/* ------------------------------------------------------------------------ */
/* RNG: hop seeds (numpy SeedSequence restated), Philox4x32-10, query keys   */
/* ------------------------------------------------------------------------ */

/* numpy.random.SeedSequence (bit_generator.pyx: _coerce_to_uint32_array,
 * mix_entropy, generate_state) -- the algorithm behind hop_seed,
 * sampling.py:135-137.  Pool size 4, 32-bit words. */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u
#define SS_XSHIFT 16

static uint32_t ss_hashmix(uint32_t value, uint32_t* hc) {
  value ^= *hc;
  *hc *= SS_MULT_A;
  value *= *hc;
  value ^= value >> SS_XSHIFT;
  return value;
}
static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> SS_XSHIFT;
  return r;
}
static int ss_words(uint64_t v, uint32_t* out) {
  /* _int_to_uint32_array: 0 -> [0]; else little-endian 32-bit words */
  int n = 0;
  if (v == 0) { out[n++] = 0; return n; }
  while (v) { out[n++] = (uint32_t)v; v >>= 32; }
  return n;
}

uint64_t or_hop_seed(uint64_t seed, uint64_t hop) {
  uint32_t ent[8];
  int ne = ss_words(seed, ent);
  ne += ss_words(hop, ent + ne);
  uint32_t pool[4];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < ne ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = 4; s < ne; s++)
    for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
  uint32_t st[2];
  uint32_t hb = SS_INIT_B;
  for (int i = 0; i < 2; i++) {
    uint32_t x = pool[i % 4];
    x ^= hb;
    hb *= SS_MULT_B;
    x *= hb;
    x ^= x >> SS_XSHIFT;
    st[i] = x;
  }
  return (uint64_t)st[0] | ((uint64_t)st[1] << 32);
}

void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

#define GF_PHILOX_TAG 0x47464232u /* "GFB2" */

/* d-th 64-bit draw of the stream keyed by (seed, query key) */
static uint64_t rand64(uint64_t seed, uint64_t qkey, uint64_t d) {
  uint32_t ctr[4] = {(uint32_t)(d >> 1), (uint32_t)qkey, (uint32_t)(qkey >> 32), GF_PHILOX_TAG};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  or_philox4x32_10(ctr, key, o);
  return (d & 1) ? ((uint64_t)o[2] | ((uint64_t)o[3] << 32)) : ((uint64_t)o[0] | ((uint64_t)o[1] << 32));
}

/* uniform integer in [0, range) by 64x64->128 multiply-high */
static uint64_t bounded(uint64_t r, uint64_t range) {
  return (uint64_t)(((unsigned __int128)r * range) >> 64);
}

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t or_child_key(uint64_t parent, uint64_t j) {
  return splitmix64(parent ^ (0x9E3779B97F4A7C15ull * (j + 1)));
}

/* ------------------------------------------------------------------------ */
/* Sampling                                                                 */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t* nbr;
  int64_t* eid;
  int64_t* ts;
  int64_t n, alloc;
} cand_buf;

static void cand_push(cand_buf* c, int64_t nbr, int64_t eid, int64_t ts) {
  if (c->n == c->alloc) {
    c->alloc = c->alloc ? c->alloc * 2 : 64;
    c->nbr = xrealloc(c->nbr, c->alloc * 8);
    c->eid = xrealloc(c->eid, c->alloc * 8);
    c->ts = xrealloc(c->ts, c->alloc * 8);
  }
  c->nbr[c->n] = nbr;
  c->eid[c->n] = eid;
  c->ts[c->n] = ts;
  c->n++;
}

/* left searchsorted over ts[0..n) */
static int64_t lower_bound(const int64_t* a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t m = lo + (hi - lo) / 2;
    if (a[m] < x) lo = m + 1; else hi = m;
  }
  return lo;
}

/* _collect_candidates, sampling.py:145-182: chronological valid candidates.
 * Returns 0 when the node is unknown/deleted (reference returns None). */
static int collect_candidates(const or_graph* g, int64_t node, int64_t t_start, int64_t t_end,
                              cand_buf* out) {
  out->n = 0;
  if (!(node >= 0 && node < g->n_nodes) || !g->node_valid[node]) return 0; /* :153-155 */
  /* walk tail -> prev, newest block first (:157-172) */
  int64_t nr = 0, ra = 16;
  int64_t* rh = (int64_t*)malloc(ra * 8 * 3);
  for (int64_t h = g->tail[node]; h != NO_BLOCK;) {
    if (t_end < g->tmin[h]) { h = g->prev[h]; continue; }
    if (t_start > g->tmax[h]) break;
    int64_t s = g->size[h];
    int64_t lo = lower_bound(g->edges[h].ts, s, t_start);
    int64_t hi = lower_bound(g->edges[h].ts, s, t_end);
    if (hi > lo) {
      if (nr == ra) { ra *= 2; rh = xrealloc(rh, ra * 8 * 3); }
      rh[3 * nr] = h; rh[3 * nr + 1] = lo; rh[3 * nr + 2] = hi;
      nr++;
    }
    h = g->prev[h];
  }
  for (int64_t r = nr - 1; r >= 0; r--) { /* oldest block first (:176-181) */
    int64_t h = rh[3 * r], lo = rh[3 * r + 1], hi = rh[3 * r + 2];
    const or_edges* e = &g->edges[h];
    for (int64_t i = lo; i < hi; i++)
      if (e->valid[i] && g->node_valid[e->nbr[i]]) cand_push(out, e->nbr[i], e->eid[i], e->ts[i]);
  }
  free(rh);
  return 1;
}

/* Floyd's k-of-n selection driven by the Philox stream; sel[] gets k
 * candidate indices in generation order.  Requires k < n. */
static void floyd_select(int64_t n, int64_t k, uint64_t seed, uint64_t qkey, int64_t* sel) {
  int64_t m = 0;
  for (int64_t j = n - k; j < n; j++) {
    int64_t t = (int64_t)bounded(rand64(seed, qkey, (uint64_t)(j - (n - k))), (uint64_t)(j + 1));
    int dup = 0;
    for (int64_t q = 0; q < m; q++)
      if (sel[q] == t) { dup = 1; break; }
    sel[m++] = dup ? j : t;
  }
}

/* _sample_one + _select, sampling.py:185-216 (uniform: see header note).
 * Faithful path: materialise all candidates like the reference. */
static int64_t sample_one_faithful(const or_graph* g, int64_t node, int64_t t_start,
                                   int64_t t_end, int64_t fanout, int policy, int64_t delta,
                                   uint64_t seed, uint64_t qkey, cand_buf* cb, int64_t* sel,
                                   int64_t* o_nbr, int64_t* o_eid, int64_t* o_ts, int write) {
  if (policy == OR_TIME_WINDOW) { /* :202-203 */
    t_start = (t_end < TS_MIN + delta) ? TS_MIN : t_end - delta;
  }
  if (!collect_candidates(g, node, t_start, t_end, cb)) return 0;
  int64_t n = cb->n;
  if (n == 0) return 0;
  int64_t k = fanout < n ? fanout : n;
  if (!write) return k;
  if (policy == OR_RECENT || k == n) { /* newest first (:188-190) */
    for (int64_t i = 0; i < k; i++) {
      o_nbr[i] = cb->nbr[n - 1 - i];
      o_eid[i] = cb->eid[n - 1 - i];
      o_ts[i] = cb->ts[n - 1 - i];
    }
    return k;
  }
  floyd_select(n, k, seed, qkey, sel);
  for (int64_t i = 0; i < k; i++) {
    o_nbr[i] = cb->nbr[sel[i]];
    o_eid[i] = cb->eid[sel[i]];
    o_ts[i] = cb->ts[sel[i]];
  }
  return k;
}

/* General-path uniform selection (graphs with deletions): see sample_one_fast */
#define OR_GEN_EXACT 64
#define OR_KREJ 32
#define OR_KFLOYD 16 /* KMAX: fanouts served by the fused kernels */
#define OR_REJ_TAG (1ull << 31) /* Philox block 2^30 + d/2: disjoint from the Floyd draws */

/* Early-exit path, same output: position-indexed view of the node list. */
typedef struct {
  int64_t nb;
  int64_t* h; /* handles head..tail */
  int64_t* cum; /* list position of each block's first slot */
} node_view;

static int64_t nv_lower_bound(const or_graph* g, const node_view* v, int64_t x) {
  /* number of list slots with ts < x (ts non-decreasing along the list) */
  int64_t lo = 0, hi = v->nb; /* find last block with tmin < x */
  while (lo < hi) {
    int64_t m = (lo + hi) / 2;
    if (g->tmin[v->h[m]] < x) lo = m + 1; else hi = m;
  }
  if (lo == 0) return 0;
  int64_t b = lo - 1, h = v->h[b];
  return v->cum[b] + lower_bound(g->edges[h].ts, g->size[h], x);
}

static void nv_at(const or_graph* g, const node_view* v, int64_t pos, int64_t* h, int64_t* i) {
  int64_t lo = 0, hi = v->nb; /* last block with cum <= pos */
  while (hi - lo > 1) {
    int64_t m = (lo + hi) / 2;
    if (v->cum[m] <= pos) lo = m; else hi = m;
  }
  *h = v->h[lo];
  *i = pos - v->cum[lo];
}

static int64_t sample_one_fast(const or_graph* g, int64_t node, int64_t t_start, int64_t t_end,
                               int64_t fanout, int policy, int64_t delta, uint64_t seed,
                               uint64_t qkey, node_view* nv, int64_t* sel, int64_t** scratch,
                               int64_t* scratch_n, int64_t* o_nbr, int64_t* o_eid, int64_t* o_ts,
                               int write, int any_deleted) {
  if (policy == OR_TIME_WINDOW) t_start = (t_end < TS_MIN + delta) ? TS_MIN : t_end - delta;
  if (!(node >= 0 && node < g->n_nodes) || !g->node_valid[node]) return 0;
  /* build the node's block directory */
  nv->nb = 0;
  int64_t acc = 0;
  for (int64_t h = g->head[node]; h != NO_BLOCK; h = g->next[h]) {
    if (nv->nb % 64 == 0) {
      nv->h = xrealloc(nv->h, (nv->nb + 64) * 8);
      nv->cum = xrealloc(nv->cum, (nv->nb + 64) * 8);
    }
    nv->h[nv->nb] = h;
    nv->cum[nv->nb] = acc;
    acc += g->size[h];
    nv->nb++;
  }
  if (nv->nb == 0) return 0;
  int64_t lo = (t_start == TS_MIN) ? 0 : nv_lower_bound(g, nv, t_start);
  int64_t hi = nv_lower_bound(g, nv, t_end);
  if (hi <= lo) return 0;
  if (!any_deleted) {
    int64_t n = hi - lo, k = fanout < n ? fanout : n;
    if (!write) return k;
    for (int64_t i = 0; i < k; i++) {
      int64_t p;
      if (policy == OR_RECENT || k == n) p = hi - 1 - i;
      else {
        if (i == 0) floyd_select(n, k, seed, qkey, sel);
        p = lo + sel[i];
      }
      int64_t h, j;
      nv_at(g, nv, p, &h, &j);
      o_nbr[i] = g->edges[h].nbr[j];
      o_eid[i] = g->edges[h].eid[j];
      o_ts[i] = g->edges[h].ts[j];
    }
    return k;
  }
  /* with deletions, uniform / time-window over a window of more than GEN_EXACT positions: draw
   * positions (Philox draws REJ_TAG + d), keep a draw whose candidate is valid and new, stop at
   * fanout keeps -- a uniform k-subset of the valid candidates (the CUDA general path,
   * gf_sample.cu k_count_general, makes the same decisions in the same draw order).  After
   * 8 * fanout + 32 draws without fanout keeps, the exact path below runs. */
  /* First (fanouts up to OR_KFLOYD, the CUDA fused kernel k_sample_fused_del): Floyd's k distinct
   * positions of the window -- the draws of the no-deletion path -- and the valid ones are kept in
   * draw order (a query no deletion touches keeps its pre-deletion sample).  They are a uniform
   * subset of the valid candidates of a uniform size; the draws below top them up with uniform new
   * valid candidates, so the result stays a uniform k-subset. */
  if (policy != OR_RECENT && hi - lo > OR_GEN_EXACT && fanout <= OR_KREJ) {
    int64_t npos = hi - lo, dmax = 8 * fanout + 32, acc = 0;
    if (fanout <= OR_KFLOYD) {
      int64_t fl[OR_KFLOYD];
      floyd_select(npos, fanout, seed, qkey, fl);
      for (int64_t i = 0; i < fanout; i++) {
        int64_t h, j;
        nv_at(g, nv, lo + fl[i], &h, &j);
        const or_edges* e = &g->edges[h];
        if (e->valid[j] && g->node_valid[e->nbr[j]]) sel[acc++] = lo + fl[i];
      }
    }
    for (int64_t d = 0; d < dmax && acc < fanout; d++) {
      int64_t p = lo + (int64_t)bounded(rand64(seed, qkey, OR_REJ_TAG + (uint64_t)d), (uint64_t)npos);
      int64_t h, j;
      nv_at(g, nv, p, &h, &j);
      const or_edges* e = &g->edges[h];
      if (!(e->valid[j] && g->node_valid[e->nbr[j]])) continue;
      int dup = 0;
      for (int64_t q = 0; q < acc; q++)
        if (sel[q] == p) { dup = 1; break; }
      if (!dup) sel[acc++] = p;
    }
    if (acc == fanout) {
      if (!write) return fanout;
      for (int64_t i = 0; i < fanout; i++) {
        int64_t h, j;
        nv_at(g, nv, sel[i], &h, &j);
        o_nbr[i] = g->edges[h].nbr[j];
        o_eid[i] = g->edges[h].eid[j];
        o_ts[i] = g->edges[h].ts[j];
      }
      return fanout;
    }
  }
  /* with deletions: list the valid positions (newest first) */
  int64_t nv_n = 0;
  int64_t need = (policy == OR_RECENT) ? fanout : (hi - lo);
  for (int64_t p = hi - 1; p >= lo && nv_n < need; p--) {
    int64_t h, j;
    nv_at(g, nv, p, &h, &j);
    const or_edges* e = &g->edges[h];
    if (e->valid[j] && g->node_valid[e->nbr[j]]) {
      if (nv_n == *scratch_n) {
        *scratch_n = *scratch_n ? *scratch_n * 2 : 256;
        *scratch = xrealloc(*scratch, *scratch_n * 8);
      }
      (*scratch)[nv_n++] = p;
    }
  }
  int64_t n = nv_n; /* for uniform: all valid candidates */
  int64_t k = fanout < n ? fanout : n;
  if (!write) return k;
  for (int64_t i = 0; i < k; i++) {
    int64_t p;
    if (policy == OR_RECENT || k == n) p = (*scratch)[i];
    else {
      if (i == 0) floyd_select(n, k, seed, qkey, sel);
      p = (*scratch)[n - 1 - sel[i]]; /* candidate index c is chronological rank */
    }
    int64_t h, j;
    nv_at(g, nv, p, &h, &j);
    o_nbr[i] = g->edges[h].nbr[j];
    o_eid[i] = g->edges[h].eid[j];
    o_ts[i] = g->edges[h].ts[j];
  }
  return k;
}

typedef struct {
  const or_graph* g;
  const int64_t *src, *t_start, *t_end;
  int64_t lo_q, hi_q;
  int64_t fanout;
  int policy;
  int64_t delta;
  uint64_t seed;
  const uint64_t* keys;
  int64_t* counts; /* pass 1 out */
  int64_t* offsets; /* pass 2 in */
  int64_t *o_nbr, *o_eid, *o_ts;
  int64_t out_cap;
  int pass, faithful, any_deleted;
} sl_task;

static void* sl_worker(void* arg) {
  sl_task* t = (sl_task*)arg;
  cand_buf cb = {0};
  node_view nv = {0};
  int64_t* scratch = NULL;
  int64_t scratch_n = 0;
  int64_t sel_n = t->fanout < 4096 ? t->fanout : 4096;
  int64_t* sel = (int64_t*)malloc((sel_n > 0 ? sel_n : 1) * 8);
  int64_t* tmp_n = NULL, *tmp_e = NULL, *tmp_t = NULL;
  int64_t tmp_cap = 0;
  for (int64_t q = t->lo_q; q < t->hi_q; q++) {
    uint64_t key = t->keys ? t->keys[q] : (uint64_t)q;
    int write = (t->pass == 2);
    int64_t *on = NULL, *oe = NULL, *ot = NULL;
    int64_t k_expect = 0;
    if (write) {
      k_expect = t->offsets[q + 1] - t->offsets[q];
      if (k_expect == 0) continue;
      if (t->offsets[q + 1] <= t->out_cap) {
        on = t->o_nbr + t->offsets[q];
        oe = t->o_eid + t->offsets[q];
        ot = t->o_ts + t->offsets[q];
      } else {
        if (tmp_cap < k_expect) {
          tmp_cap = k_expect;
          tmp_n = xrealloc(tmp_n, tmp_cap * 8);
          tmp_e = xrealloc(tmp_e, tmp_cap * 8);
          tmp_t = xrealloc(tmp_t, tmp_cap * 8);
        }
        on = tmp_n; oe = tmp_e; ot = tmp_t;
      }
      if (t->fanout > sel_n && k_expect > sel_n) {
        sel_n = k_expect;
        sel = xrealloc(sel, sel_n * 8);
      }
    }
    int64_t k;
    /* with deletions the uniform / time-window selection is position-based (rejection draws over
     * the window, see sample_one_fast), so it runs on the position-indexed view in both modes */
    if (t->faithful && !(t->any_deleted && t->policy != OR_RECENT))
      k = sample_one_faithful(t->g, t->src[q], t->t_start[q], t->t_end[q], t->fanout, t->policy,
                              t->delta, t->seed, key, &cb, sel, on, oe, ot, write);
    else
      k = sample_one_fast(t->g, t->src[q], t->t_start[q], t->t_end[q], t->fanout, t->policy,
                          t->delta, t->seed, key, &nv, sel, &scratch, &scratch_n, on, oe, ot,
                          write, t->any_deleted);
    if (!write) t->counts[q] = k;
    else if (on == tmp_n && on) { /* partial copy up to out_cap */
      for (int64_t i = 0; i < k; i++) {
        int64_t p = t->offsets[q] + i;
        if (p < t->out_cap) { t->o_nbr[p] = on[i]; t->o_eid[p] = oe[i]; t->o_ts[p] = ot[i]; }
      }
    }
  }
  free(cb.nbr); free(cb.eid); free(cb.ts);
  free(nv.h); free(nv.cum);
  free(scratch); free(sel);
  free(tmp_n); free(tmp_e); free(tmp_t);
  return NULL;
}

static int graph_any_deleted(const or_graph* g) {
  for (int64_t v = 0; v < g->n_nodes; v++)
    if (!g->node_valid[v]) return 1;
  for (int64_t v = 0; v < g->n_nodes; v++) {
    int64_t live = 0;
    for (int64_t h = g->head[v]; h != NO_BLOCK; h = g->next[h]) live += g->size[h];
    if (live != g->degree[v]) return 1;
  }
  return 0;
}

static void run_pass(sl_task* base, int64_t n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > n) threads = (int)(n > 0 ? n : 1);
  pthread_t* th = (pthread_t*)malloc(threads * sizeof(pthread_t));
  sl_task* ts = (sl_task*)malloc(threads * sizeof(sl_task));
  for (int i = 0; i < threads; i++) {
    ts[i] = *base;
    ts[i].lo_q = n * i / threads;
    ts[i].hi_q = n * (i + 1) / threads;
    if (threads > 1) pthread_create(&th[i], NULL, sl_worker, &ts[i]);
  }
  if (threads == 1) sl_worker(&ts[0]);
  else for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
  free(th);
  free(ts);
}

int64_t or_sample_layer(const or_graph* g, const int64_t* src, const int64_t* t_start,
                        const int64_t* t_end, int64_t n, int64_t fanout, int policy, int64_t delta,
                        uint64_t seed, const uint64_t* keys, int64_t* offsets, int64_t* out_nbr,
                        int64_t* out_eid, int64_t* out_ts, int64_t out_cap, int threads,
                        int faithful) {
  if (fanout < 1 || n < 0) return -1; /* :238-241 */
  if (policy < 0 || policy > 2) return -1;
  if (policy == OR_TIME_WINDOW && delta <= 0) return -1;
  sl_task base;
  memset(&base, 0, sizeof(base));
  base.g = g; base.src = src; base.t_start = t_start; base.t_end = t_end;
  base.fanout = fanout; base.policy = policy; base.delta = delta; base.seed = seed;
  base.keys = keys; base.faithful = faithful;
  base.any_deleted = graph_any_deleted(g);
  base.counts = offsets + 1;
  base.pass = 1;
  offsets[0] = 0;
  run_pass(&base, n, threads);
  for (int64_t i = 0; i < n; i++) offsets[i + 1] += offsets[i]; /* :262-264 */
  base.offsets = offsets;
  base.o_nbr = out_nbr; base.o_eid = out_eid; base.o_ts = out_ts; base.out_cap = out_cap;
  base.pass = 2;
  run_pass(&base, n, threads);
  return offsets[n];
}

int or_sample_khop(const or_graph* g, const int64_t* roots, const int64_t* ts, int64_t n_roots,
                   const int64_t* fanouts, int n_hops, int policy, int64_t delta, uint64_t seed,
                   uint64_t root_key_base, int64_t** offsets, int64_t** out_nbr,
                   int64_t** out_eid, int64_t** out_ts, const int64_t* caps, int64_t* totals,
                   int threads, int faithful) {
  /* sampling.py:276-299: hop l uses (prev neighbors, TS_MIN, prev timestamps) */
  for (int h = 0; h < n_hops; h++)
    if (fanouts[h] < 1) return -1;
  int64_t n = n_roots;
  const int64_t* srcs = roots;
  const int64_t* tends = ts;
  uint64_t* keys = (uint64_t*)malloc((n > 0 ? n : 1) * 8);
  for (int64_t i = 0; i < n; i++) keys[i] = root_key_base + (uint64_t)i;
  int rc = 0;
  for (int h = 0; h < n_hops; h++) {
    int64_t* tstart = (int64_t*)malloc((n > 0 ? n : 1) * 8);
    for (int64_t i = 0; i < n; i++) tstart[i] = TS_MIN;
    int64_t tot = or_sample_layer(g, srcs, tstart, tends, n, fanouts[h], policy, delta,
                                  or_hop_seed(seed, (uint64_t)h), keys, offsets[h], out_nbr[h],
                                  out_eid[h], out_ts[h], caps[h], threads, faithful);
    free(tstart);
    totals[h] = tot;
    if (tot < 0) { rc = -1; break; }
    if (tot > caps[h]) { rc = -2; break; }
    uint64_t* nk = (uint64_t*)malloc((tot > 0 ? tot : 1) * 8);
    for (int64_t i = 0; i < n; i++)
      for (int64_t p = offsets[h][i]; p < offsets[h][i + 1]; p++)
        nk[p] = or_child_key(keys[i], (uint64_t)(p - offsets[h][i]));
    free(keys);
    keys = nk;
    srcs = out_nbr[h];
    tends = out_ts[h];
    n = tot;
  }
  free(keys);
  return rc;
}
