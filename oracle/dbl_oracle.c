/*
 * dbl_oracle.c -- CPU restatement of the dblreach reference algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker the CUDA engine is
 * compared against and the "port" CPU baseline that bench.py times; it is
 * never linked into, loaded by, or called from the product path
 * (paper_2101_09441_b200/).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/dblreach/):
 *
 *   orc_leaf_hash        labels.py:119-137   splitmix64 mix mod k'
 *   orc_graph_*          graph.py:31-66      adjacency lists in insertion
 *                                            order, duplicate edges dropped
 *   orc_select_landmarks labels.py:140-147   top-k by (-score, id)
 *   orc_select_leaves    labels.py:150-181   zero in/out degree (+ M(v)<=r)
 *   orc_build            labels.py:247-306   one _flood BFS per landmark bit
 *                                            and per occupied bucket
 *   orc_query_batch      queries.py:94-142, 210-249  rules 0..4 then the
 *                                            pruned BFS; contiguous slices
 *                                            per worker thread
 *   orc_insert_edge      updates.py:89-137   pre-check, add_edge, pruned
 *                                            union propagation both ways
 *   orc_reach            graph.py:245-263    plain BFS ground truth
 *
 * Parity pin: tests/test_oracle.py checks this file against the golden
 * vectors produced by oracle/gen_golden.py, which runs the reference itself.
 *
 * Bit order follows pkg/docs/snapshot-format.md:38-42: bit i of a label is
 * bit (i % 64) of word (i / 64).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_OK 0
#define ORC_E_RANGE 1
#define ORC_E_CONFIG 2
#define ORC_E_MISMATCH 3
#define ORC_E_OOM 6

/* ---------------------------------------------------------------- hash -- */

uint32_t orc_leaf_hash(uint64_t v, uint32_t k_prime, uint64_t seed) {
    /* labels.py:131-137; all arithmetic mod 2^64 */
    uint64_t x = v * 0x9E3779B97F4A7C15ULL + seed * 0xD1B54A32D192ED03ULL;
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ULL;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBULL;
    x ^= x >> 31;
    return (uint32_t)(x % (uint64_t)k_prime);
}

/* --------------------------------------------------------------- graph -- */

typedef struct {
    uint32_t *a;
    uint32_t len, cap;
} orc_vec;

typedef struct {
    uint32_t n;
    uint64_t m;
    orc_vec *fwd, *rev;
    /* open-addressing edge set, graph.py:41,60-61 */
    uint64_t *keys;
    uint64_t cap;
} orc_graph;

static int vec_push(orc_vec *v, uint32_t x) {
    if (v->len == v->cap) {
        uint32_t nc = v->cap ? v->cap * 2 : 4;
        uint32_t *na = (uint32_t *)realloc(v->a, (size_t)nc * sizeof(uint32_t));
        if (!na) return ORC_E_OOM;
        v->a = na;
        v->cap = nc;
    }
    v->a[v->len++] = x;
    return ORC_OK;
}

static inline uint64_t mix64(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

#define EMPTY_KEY 0xFFFFFFFFFFFFFFFFULL

static int set_grow(orc_graph *g) {
    uint64_t nc = g->cap ? g->cap * 2 : 1024;
    uint64_t *nk = (uint64_t *)malloc(nc * sizeof(uint64_t));
    if (!nk) return ORC_E_OOM;
    memset(nk, 0xFF, nc * sizeof(uint64_t));
    for (uint64_t i = 0; i < g->cap; ++i) {
        uint64_t k = g->keys[i];
        if (k == EMPTY_KEY) continue;
        uint64_t h = mix64(k) & (nc - 1);
        while (nk[h] != EMPTY_KEY) h = (h + 1) & (nc - 1);
        nk[h] = k;
    }
    free(g->keys);
    g->keys = nk;
    g->cap = nc;
    return ORC_OK;
}

/* returns 1 if inserted, 0 if present */
static int set_insert(orc_graph *g, uint64_t key) {
    if ((g->m + 1) * 2 > g->cap) {
        if (set_grow(g)) return -1;
    }
    uint64_t h = mix64(key) & (g->cap - 1);
    while (g->keys[h] != EMPTY_KEY) {
        if (g->keys[h] == key) return 0;
        h = (h + 1) & (g->cap - 1);
    }
    g->keys[h] = key;
    return 1;
}

static int set_has(const orc_graph *g, uint64_t key) {
    if (!g->cap) return 0;
    uint64_t h = mix64(key) & (g->cap - 1);
    while (g->keys[h] != EMPTY_KEY) {
        if (g->keys[h] == key) return 1;
        h = (h + 1) & (g->cap - 1);
    }
    return 0;
}

void orc_graph_free(orc_graph *g) {
    if (!g) return;
    if (g->fwd) for (uint32_t i = 0; i < g->n; ++i) free(g->fwd[i].a);
    if (g->rev) for (uint32_t i = 0; i < g->n; ++i) free(g->rev[i].a);
    free(g->fwd);
    free(g->rev);
    free(g->keys);
    free(g);
}

orc_graph *orc_graph_new(uint32_t n) {
    orc_graph *g = (orc_graph *)calloc(1, sizeof(orc_graph));
    if (!g) return NULL;
    g->n = n;
    g->fwd = (orc_vec *)calloc(n ? n : 1, sizeof(orc_vec));
    g->rev = (orc_vec *)calloc(n ? n : 1, sizeof(orc_vec));
    if (!g->fwd || !g->rev) { orc_graph_free(g); return NULL; }
    return g;
}

/* DynamicGraph.add_edge, graph.py:56-66.  Returns 1 new, 0 dup, <0 error. */
int orc_graph_add_edge(orc_graph *g, uint32_t u, uint32_t v) {
    if (u >= g->n || v >= g->n) return -ORC_E_RANGE;
    int r = set_insert(g, ((uint64_t)u << 32) | v);
    if (r < 0) return -ORC_E_OOM;
    if (r == 0) return 0;
    if (vec_push(&g->fwd[u], v) || vec_push(&g->rev[v], u)) return -ORC_E_OOM;
    g->m++;
    return 1;
}

int orc_graph_add_edges(orc_graph *g, const uint32_t *src, const uint32_t *dst, uint64_t m) {
    for (uint64_t i = 0; i < m; ++i) {
        int r = orc_graph_add_edge(g, src[i], dst[i]);
        if (r < 0) return -r;
    }
    return ORC_OK;
}

uint64_t orc_graph_edge_count(const orc_graph *g) { return g->m; }
int orc_graph_has_edge(const orc_graph *g, uint32_t u, uint32_t v) {
    return set_has(g, ((uint64_t)u << 32) | v);
}

void orc_graph_degrees(const orc_graph *g, uint32_t *indeg, uint32_t *outdeg) {
    for (uint32_t v = 0; v < g->n; ++v) {
        indeg[v] = g->rev[v].len;
        outdeg[v] = g->fwd[v].len;
    }
}

/* ----------------------------------------------------------- metadata -- */

/* LandmarkStrategy.score, labels.py:39-46: 0=max 1=min 2=sum 3=product */
static inline uint64_t strat_score(int s, uint64_t in, uint64_t out) {
    switch (s) {
    case 0: return in > out ? in : out;
    case 1: return in < out ? in : out;
    case 2: return in + out;
    default: return in * out;
    }
}

typedef struct { uint64_t score; uint32_t id; } scored;

static int cmp_scored(const void *a, const void *b) {
    const scored *x = (const scored *)a, *y = (const scored *)b;
    if (x->score != y->score) return x->score > y->score ? -1 : 1; /* -score */
    return x->id < y->id ? -1 : (x->id > y->id);                    /* then id */
}

/* select_landmarks, labels.py:140-147 */
int orc_select_landmarks(const orc_graph *g, uint32_t k, int strategy, uint32_t *out) {
    if (k > g->n) return ORC_E_CONFIG;
    scored *s = (scored *)malloc((size_t)(g->n ? g->n : 1) * sizeof(scored));
    if (!s) return ORC_E_OOM;
    for (uint32_t v = 0; v < g->n; ++v) {
        s[v].score = strat_score(strategy, g->rev[v].len, g->fwd[v].len);
        s[v].id = v;
    }
    qsort(s, g->n, sizeof(scored), cmp_scored);
    for (uint32_t i = 0; i < k; ++i) out[i] = s[i].id;
    free(s);
    return ORC_OK;
}

/* select_leaves, labels.py:150-181.  flags bit0 = source leaf (leaves_in),
 * bit1 = sink leaf (leaves_out); bucket[v] valid where flags != 0.
 * ovr_bucket[v] < k_prime overrides leaf_hash (0xFFFFFFFF = none). */
int orc_select_leaves(const orc_graph *g, uint64_t threshold, uint32_t k_prime,
                      uint64_t seed, const uint32_t *ovr_bucket,
                      uint8_t *flags, uint32_t *bucket) {
    if (k_prime < 1) return ORC_E_CONFIG;
    for (uint32_t v = 0; v < g->n; ++v) {
        uint64_t in = g->rev[v].len, out = g->fwd[v].len;
        uint8_t f = 0;
        if (in == 0) f |= 1;
        if (out == 0) f |= 2;
        if (threshold > 0 && in * out <= threshold) f |= 3;
        flags[v] = f;
        bucket[v] = 0;
        if (f) {
            if (ovr_bucket && ovr_bucket[v] != 0xFFFFFFFFu) {
                if (ovr_bucket[v] >= k_prime) return ORC_E_CONFIG;
                bucket[v] = ovr_bucket[v];
            } else {
                bucket[v] = orc_leaf_hash(v, k_prime, seed);
            }
        }
    }
    return ORC_OK;
}

/* -------------------------------------------------------------- build -- */

/* _flood, labels.py:247-260.  Word array `lab` has `stride` words per
 * vertex; the flooded bit is (word w, mask bit).  Uses relaxed atomics so
 * threads flooding different bits of one word can run concurrently. */
static void flood(orc_vec *adj, const uint32_t *seeds, uint32_t nseeds,
                  uint64_t *lab, uint32_t stride, uint32_t w, uint64_t bit,
                  uint32_t *queue) {
    uint32_t head = 0, tail = 0;
    for (uint32_t i = 0; i < nseeds; ++i) {
        uint32_t s = seeds[i];
        uint64_t *p = &lab[(uint64_t)s * stride + w];
        if (!(__atomic_load_n(p, __ATOMIC_RELAXED) & bit)) {
            __atomic_fetch_or(p, bit, __ATOMIC_RELAXED);
            queue[tail++] = s;
        }
    }
    while (head < tail) {
        uint32_t pv = queue[head++];
        const orc_vec *a = &adj[pv];
        for (uint32_t j = 0; j < a->len; ++j) {
            uint32_t x = a->a[j];
            uint64_t *q = &lab[(uint64_t)x * stride + w];
            if (!(__atomic_load_n(q, __ATOMIC_RELAXED) & bit)) {
                __atomic_fetch_or(q, bit, __ATOMIC_RELAXED);
                queue[tail++] = x;
            }
        }
    }
}

typedef struct {
    const orc_graph *g;
    uint32_t k, kp, wdl, wbl;
    const uint32_t *landmarks;
    /* bucket seeds: CSR over buckets, separately for in and out */
    const uint32_t *bin_off, *bin_ids, *bout_off, *bout_ids;
    uint64_t *dl_in, *dl_out, *bl_in, *bl_out;
    uint32_t ntasks;
    uint32_t next; /* atomic task counter */
    int err;
} build_ctx;

static void *build_worker(void *arg) {
    build_ctx *c = (build_ctx *)arg;
    uint32_t *queue = (uint32_t *)malloc((size_t)(c->g->n ? c->g->n : 1) * sizeof(uint32_t));
    if (!queue) { c->err = ORC_E_OOM; return NULL; }
    for (;;) {
        uint32_t t = __atomic_fetch_add(&c->next, 1, __ATOMIC_RELAXED);
        if (t >= c->ntasks) break;
        /* task order: landmark i fwd, landmark i rev, bucket b in, bucket b out */
        if (t < 2 * c->k) {
            uint32_t i = t / 2;
            uint32_t l = c->landmarks[i];
            if (t % 2 == 0)
                flood(c->g->fwd, &l, 1, c->dl_in, c->wdl, i / 64, 1ULL << (i % 64), queue);
            else
                flood(c->g->rev, &l, 1, c->dl_out, c->wdl, i / 64, 1ULL << (i % 64), queue);
        } else {
            uint32_t r = t - 2 * c->k;
            uint32_t b = r / 2;
            if (r % 2 == 0) {
                uint32_t s0 = c->bin_off[b], s1 = c->bin_off[b + 1];
                if (s1 > s0)
                    flood(c->g->fwd, c->bin_ids + s0, s1 - s0, c->bl_in, c->wbl, b / 64,
                          1ULL << (b % 64), queue);
            } else {
                uint32_t s0 = c->bout_off[b], s1 = c->bout_off[b + 1];
                if (s1 > s0)
                    flood(c->g->rev, c->bout_ids + s0, s1 - s0, c->bl_out, c->wbl, b / 64,
                          1ULL << (b % 64), queue);
            }
        }
    }
    free(queue);
    return NULL;
}

/* build_index, labels.py:263-306, with pinned metadata (landmarks, leaf
 * flags, buckets) as produced by orc_select_* or given by the caller.
 * Label arrays are n x ceil(k/64) and n x ceil(k'/64) u64, zeroed here.
 * Floods of distinct bits are independent, so `threads` workers may run
 * them concurrently; results are identical to the sequential order. */
int orc_build(const orc_graph *g, uint32_t k, uint32_t k_prime,
              const uint32_t *landmarks, const uint8_t *leaf_flags,
              const uint32_t *bucket, uint64_t *dl_in, uint64_t *dl_out,
              uint64_t *bl_in, uint64_t *bl_out, int threads) {
    uint32_t n = g->n;
    uint32_t wdl = (k + 63) / 64, wbl = (k_prime + 63) / 64;
    if (k > n || k_prime < 1) return ORC_E_CONFIG;
    memset(dl_in, 0, (size_t)n * wdl * 8);
    memset(dl_out, 0, (size_t)n * wdl * 8);
    memset(bl_in, 0, (size_t)n * wbl * 8);
    memset(bl_out, 0, (size_t)n * wbl * 8);
    /* group leaves by bucket in ascending id order (labels.py:295-305) */
    uint32_t *bin_off = (uint32_t *)calloc(k_prime + 1, 4);
    uint32_t *bout_off = (uint32_t *)calloc(k_prime + 1, 4);
    uint32_t nin = 0, nout = 0;
    for (uint32_t v = 0; v < n; ++v) {
        if (leaf_flags[v] & 1) { bin_off[bucket[v] + 1]++; nin++; }
        if (leaf_flags[v] & 2) { bout_off[bucket[v] + 1]++; nout++; }
    }
    for (uint32_t b = 0; b < k_prime; ++b) {
        bin_off[b + 1] += bin_off[b];
        bout_off[b + 1] += bout_off[b];
    }
    uint32_t *bin_ids = (uint32_t *)malloc((size_t)(nin ? nin : 1) * 4);
    uint32_t *bout_ids = (uint32_t *)malloc((size_t)(nout ? nout : 1) * 4);
    uint32_t *fin = (uint32_t *)calloc(k_prime, 4), *fout = (uint32_t *)calloc(k_prime, 4);
    for (uint32_t v = 0; v < n; ++v) {
        if (leaf_flags[v] & 1) { uint32_t b = bucket[v]; bin_ids[bin_off[b] + fin[b]++] = v; }
        if (leaf_flags[v] & 2) { uint32_t b = bucket[v]; bout_ids[bout_off[b] + fout[b]++] = v; }
    }
    free(fin);
    free(fout);
    build_ctx c = {g, k, k_prime, wdl, wbl, landmarks, bin_off, bin_ids, bout_off,
                   bout_ids, dl_in, dl_out, bl_in, bl_out, 2 * k + 2 * k_prime, 0, 0};
    if (threads < 1) threads = 1;
    if (threads == 1) {
        build_worker(&c);
    } else {
        pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
        for (int i = 0; i < threads; ++i) pthread_create(&tid[i], NULL, build_worker, &c);
        for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
        free(tid);
    }
    free(bin_off); free(bout_off); free(bin_ids); free(bout_ids);
    return c.err;
}

/* -------------------------------------------------------------- query -- */

/* AnsweredBy order, queries.py:40-47 / _ANSWER_ORDER :188-189 */
enum { A_REFLEXIVE = 0, A_DL_POS = 1, A_BL_NEG = 2, A_THM1 = 3, A_THM2 = 4,
       A_BFS_POS = 5, A_BFS_NEG = 6 };

/* QueryFlags, queries.py:59-75, as bits */
#define F_USE_DL 1u
#define F_USE_BL 2u
#define F_THM1 4u
#define F_THM2 8u
#define F_PRUNE_DL 16u
#define F_PRUNE_BL 32u

typedef struct {
    const orc_graph *g;
    uint32_t wdl, wbl;
    const uint64_t *dl_in, *dl_out, *bl_in, *bl_out;
    const uint32_t *qu, *qv;
    uint8_t *codes;
    uint32_t *visited;
    uint32_t flags;
    uint64_t lo, hi;
    int err;
} qslice;

static inline int and_nz(const uint64_t *a, const uint64_t *b, uint32_t w) {
    for (uint32_t i = 0; i < w; ++i) if (a[i] & b[i]) return 1;
    return 0;
}
static inline int andnot_nz(const uint64_t *a, const uint64_t *b, uint32_t w) {
    for (uint32_t i = 0; i < w; ++i) if (a[i] & ~b[i]) return 1;
    return 0;
}

/* _run_slice + query, queries.py:94-142, 169-173 */
static void *query_slice(void *arg) {
    qslice *s = (qslice *)arg;
    const orc_graph *g = s->g;
    uint32_t n = g->n, wdl = s->wdl, wbl = s->wbl, fl = s->flags;
    uint32_t *stamp = (uint32_t *)calloc(n ? n : 1, 4);   /* _Scratch, :78-85 */
    uint32_t *queue = (uint32_t *)malloc((size_t)(n ? n : 1) * 4);
    uint32_t epoch = 0;
    int use_dl = !!(fl & F_USE_DL), use_bl = !!(fl & F_USE_BL);
    int prune_dl = use_dl && (fl & F_PRUNE_DL), prune_bl = use_bl && (fl & F_PRUNE_BL);
    for (uint64_t q = s->lo; q < s->hi; ++q) {
        uint32_t u = s->qu[q], v = s->qv[q];
        uint32_t vis = 0;
        uint8_t code;
        if (u >= n || v >= n) { s->err = ORC_E_RANGE; break; }
        const uint64_t *dlo_u = s->dl_out + (uint64_t)u * wdl, *dli_u = s->dl_in + (uint64_t)u * wdl;
        const uint64_t *dlo_v = s->dl_out + (uint64_t)v * wdl, *dli_v = s->dl_in + (uint64_t)v * wdl;
        const uint64_t *bli_u = s->bl_in + (uint64_t)u * wbl, *blo_u = s->bl_out + (uint64_t)u * wbl;
        const uint64_t *bli_v = s->bl_in + (uint64_t)v * wbl, *blo_v = s->bl_out + (uint64_t)v * wbl;
        if (u == v) code = A_REFLEXIVE;
        else if (use_dl && and_nz(dlo_u, dli_v, wdl)) code = A_DL_POS;
        else if (use_bl && (andnot_nz(bli_u, bli_v, wbl) || andnot_nz(blo_v, blo_u, wbl))) code = A_BL_NEG;
        else if (use_dl && (fl & F_THM1) && and_nz(dlo_v, dli_u, wdl)) code = A_THM1;
        else if (use_dl && (fl & F_THM2) && (and_nz(dlo_u, dli_u, wdl) || and_nz(dlo_v, dli_v, wdl))) code = A_THM2;
        else {
            /* pruned BFS, queries.py:116-142 */
            if (++epoch == 0) { memset(stamp, 0, (size_t)n * 4); epoch = 1; }
            stamp[u] = epoch;
            uint32_t head = 0, tail = 0;
            queue[tail++] = u;
            code = A_BFS_NEG;
            while (head < tail && code == A_BFS_NEG) {
                uint32_t w = queue[head++];
                vis++;
                const orc_vec *a = &g->fwd[w];
                for (uint32_t j = 0; j < a->len; ++j) {
                    uint32_t x = a->a[j];
                    if (x == v) { code = A_BFS_POS; break; }
                    if (stamp[x] == epoch) continue;
                    stamp[x] = epoch;
                    if (prune_dl && and_nz(dlo_u, s->dl_in + (uint64_t)x * wdl, wdl)) continue;
                    if (prune_bl && (andnot_nz(s->bl_in + (uint64_t)x * wbl, bli_v, wbl) ||
                                     andnot_nz(blo_v, s->bl_out + (uint64_t)x * wbl, wbl)))
                        continue;
                    queue[tail++] = x;
                }
            }
        }
        s->codes[q] = code;
        if (s->visited) s->visited[q] = vis;
    }
    free(stamp);
    free(queue);
    return NULL;
}

/* query_batch, queries.py:210-249: contiguous slices, one per worker,
 * outputs written in input order, so results are worker-count independent. */
int orc_query_batch(const orc_graph *g, uint32_t k, uint32_t k_prime,
                    const uint64_t *dl_in, const uint64_t *dl_out,
                    const uint64_t *bl_in, const uint64_t *bl_out,
                    const uint32_t *qu, const uint32_t *qv, uint64_t q,
                    uint32_t flags, uint8_t *codes, uint32_t *visited, int threads) {
    uint32_t wdl = (k + 63) / 64, wbl = (k_prime + 63) / 64;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads * 2 > q) threads = 1;
    qslice *sl = (qslice *)calloc(threads, sizeof(qslice));
    uint64_t chunk = (q + threads - 1) / threads;
    for (int i = 0; i < threads; ++i) {
        uint64_t lo = (uint64_t)i * chunk, hi = lo + chunk;
        if (lo > q) lo = q;
        if (hi > q) hi = q;
        qslice t = {g, wdl, wbl, dl_in, dl_out, bl_in, bl_out, qu, qv, codes, visited,
                    flags, lo, hi, 0};
        sl[i] = t;
    }
    if (threads == 1) {
        query_slice(&sl[0]);
    } else {
        pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
        for (int i = 0; i < threads; ++i) pthread_create(&tid[i], NULL, query_slice, &sl[i]);
        for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
        free(tid);
    }
    int err = 0;
    for (int i = 0; i < threads; ++i) if (sl[i].err) err = sl[i].err;
    free(sl);
    return err;
}

/* ------------------------------------------------------------- insert -- */

/* _propagate_union, updates.py:89-109.  Returns dequeues; *changed += hits */
static uint32_t propagate_union(orc_vec *adj, uint32_t n, uint32_t seed,
                                const uint64_t *dl_add, const uint64_t *bl_add,
                                uint64_t *dl, uint64_t *bl, uint32_t wdl, uint32_t wbl,
                                uint32_t *queue, uint32_t *changed) {
    (void)n;
    uint64_t *ds = dl + (uint64_t)seed * wdl, *bs = bl + (uint64_t)seed * wbl;
    if (andnot_nz(dl_add, ds, wdl) || andnot_nz(bl_add, bs, wbl)) {
        for (uint32_t i = 0; i < wdl; ++i) ds[i] |= dl_add[i];
        for (uint32_t i = 0; i < wbl; ++i) bs[i] |= bl_add[i];
        (*changed)++;
    }
    uint32_t head = 0, tail = 0, visited = 0;
    queue[tail++] = seed;
    while (head < tail) {
        uint32_t p = queue[head++];
        visited++;
        const orc_vec *a = &adj[p];
        for (uint32_t j = 0; j < a->len; ++j) {
            uint32_t x = a->a[j];
            uint64_t *dx = dl + (uint64_t)x * wdl, *bx = bl + (uint64_t)x * wbl;
            if (andnot_nz(dl_add, dx, wdl) || andnot_nz(bl_add, bx, wbl)) {
                for (uint32_t i = 0; i < wdl; ++i) dx[i] |= dl_add[i];
                for (uint32_t i = 0; i < wbl; ++i) bx[i] |= bl_add[i];
                (*changed)++;
                queue[tail++] = x;
            }
        }
    }
    return visited;
}

/* insert_edge, updates.py:112-137.  stats = {visited, labels_changed,
 * early_terminated}; labels are mutated in place. */
int orc_insert_edge(orc_graph *g, uint32_t k, uint32_t k_prime,
                    uint64_t *dl_in, uint64_t *dl_out, uint64_t *bl_in, uint64_t *bl_out,
                    uint32_t u, uint32_t v, uint32_t *stats) {
    uint32_t n = g->n, wdl = (k + 63) / 64, wbl = (k_prime + 63) / 64;
    if (u >= n || v >= n) return ORC_E_RANGE;
    int pre = and_nz(dl_out + (uint64_t)u * wdl, dl_in + (uint64_t)v * wdl, wdl);
    int r = orc_graph_add_edge(g, u, v);
    if (r < 0) return -r;
    stats[0] = stats[1] = stats[2] = 0;
    if (pre) { stats[2] = 1; return ORC_OK; }
    uint32_t *queue = (uint32_t *)malloc((size_t)(n ? n : 1) * 4);
    uint64_t add_d[64], add_b[64];  /* up to 4096-bit labels */
    if (wdl > 64 || wbl > 64 || !queue) { free(queue); return ORC_E_CONFIG; }
    memcpy(add_d, dl_in + (uint64_t)u * wdl, wdl * 8);
    memcpy(add_b, bl_in + (uint64_t)u * wbl, wbl * 8);
    uint32_t changed = 0;
    stats[0] += propagate_union(g->fwd, n, v, add_d, add_b, dl_in, bl_in, wdl, wbl, queue, &changed);
    memcpy(add_d, dl_out + (uint64_t)v * wdl, wdl * 8);
    memcpy(add_b, bl_out + (uint64_t)v * wbl, wbl * 8);
    stats[0] += propagate_union(g->rev, n, u, add_d, add_b, dl_out, bl_out, wdl, wbl, queue, &changed);
    stats[1] = changed;
    free(queue);
    return ORC_OK;
}

/* -------------------------------------------------------------- reach -- */

/* reachable set of u as a byte mask (graph.py:266-288 row u) */
int orc_reach_from(const orc_graph *g, uint32_t u, uint8_t *seen) {
    uint32_t n = g->n;
    if (u >= n) return ORC_E_RANGE;
    memset(seen, 0, n);
    uint32_t *queue = (uint32_t *)malloc((size_t)n * 4);
    uint32_t head = 0, tail = 0;
    seen[u] = 1;
    queue[tail++] = u;
    while (head < tail) {
        uint32_t w = queue[head++];
        const orc_vec *a = &g->fwd[w];
        for (uint32_t j = 0; j < a->len; ++j) {
            uint32_t x = a->a[j];
            if (!seen[x]) { seen[x] = 1; queue[tail++] = x; }
        }
    }
    free(queue);
    return ORC_OK;
}

/* oracle_reach for a batch of pairs (graph.py:245-263), threaded. */
typedef struct { const orc_graph *g; const uint32_t *qu, *qv; uint8_t *out; uint64_t lo, hi; } rslice;
static void *reach_slice(void *arg) {
    rslice *s = (rslice *)arg;
    uint32_t n = s->g->n;
    uint32_t *stamp = (uint32_t *)calloc(n ? n : 1, 4), *queue = (uint32_t *)malloc((size_t)(n ? n : 1) * 4);
    uint32_t epoch = 0;
    for (uint64_t q = s->lo; q < s->hi; ++q) {
        uint32_t u = s->qu[q], v = s->qv[q];
        uint8_t r = (u == v);
        if (!r) {
            ++epoch;
            stamp[u] = epoch;
            uint32_t head = 0, tail = 0;
            queue[tail++] = u;
            while (head < tail && !r) {
                uint32_t w = queue[head++];
                const orc_vec *a = &s->g->fwd[w];
                for (uint32_t j = 0; j < a->len; ++j) {
                    uint32_t x = a->a[j];
                    if (x == v) { r = 1; break; }
                    if (stamp[x] != epoch) { stamp[x] = epoch; queue[tail++] = x; }
                }
            }
        }
        s->out[q] = r;
    }
    free(stamp); free(queue);
    return NULL;
}

int orc_reach_batch(const orc_graph *g, const uint32_t *qu, const uint32_t *qv, uint64_t q,
                    uint8_t *out, int threads) {
    for (uint64_t i = 0; i < q; ++i) if (qu[i] >= g->n || qv[i] >= g->n) return ORC_E_RANGE;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > q) threads = 1;
    rslice *sl = (rslice *)calloc(threads, sizeof(rslice));
    uint64_t chunk = (q + threads - 1) / threads;
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; ++i) {
        uint64_t lo = (uint64_t)i * chunk, hi = lo + chunk;
        if (lo > q) lo = q;
        if (hi > q) hi = q;
        rslice t = {g, qu, qv, out, lo, hi};
        sl[i] = t;
        pthread_create(&tid[i], NULL, reach_slice, &sl[i]);
    }
    for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
    free(tid); free(sl);
    return ORC_OK;
}

/* ------------------------------------------------------ CSR variants -- */
/* Same algorithms over plain CSR arrays (no per-vertex vectors or edge
 * hash), for the large configs where the list form does not fit in host
 * memory.  Row order does not matter for any checked value. */

/* reached[v] = 1 iff some seed reaches v along (ptr, col) (a _flood,
 * labels.py:247-260, with a byte array as the visited mark). */
int orc_csr_flood(uint32_t n, const uint64_t *ptr, const uint32_t *col, const uint32_t *seeds,
                  uint64_t nseeds, uint8_t *reached) {
    uint32_t *queue = (uint32_t *)malloc((size_t)(n ? n : 1) * 4);
    if (!queue) return ORC_E_OOM;
    memset(reached, 0, n);
    uint64_t head = 0, tail = 0;
    for (uint64_t i = 0; i < nseeds; ++i)
        if (!reached[seeds[i]]) { reached[seeds[i]] = 1; queue[tail++] = seeds[i]; }
    while (head < tail) {
        uint32_t p = queue[head++];
        for (uint64_t e = ptr[p]; e < ptr[p + 1]; ++e) {
            uint32_t x = col[e];
            if (!reached[x]) { reached[x] = 1; queue[tail++] = x; }
        }
    }
    free(queue);
    return ORC_OK;
}

typedef struct {
    uint32_t n, wdl, wbl;
    const uint64_t *ptr;
    const uint32_t *col;
    const uint64_t *dl_in, *dl_out, *bl_in, *bl_out;
    const uint32_t *qu, *qv;
    uint8_t *codes;
    uint32_t flags;
    uint64_t lo, hi;
    int err;
} cslice;

/* query (queries.py:94-142) over a CSR forward adjacency */
static void *csr_query_slice(void *arg) {
    cslice *s = (cslice *)arg;
    uint32_t n = s->n, wdl = s->wdl, wbl = s->wbl, fl = s->flags;
    uint32_t *stamp = (uint32_t *)calloc(n ? n : 1, 4);
    uint32_t *queue = (uint32_t *)malloc((size_t)(n ? n : 1) * 4);
    uint32_t epoch = 0;
    int use_dl = !!(fl & F_USE_DL), use_bl = !!(fl & F_USE_BL);
    int prune_dl = use_dl && (fl & F_PRUNE_DL), prune_bl = use_bl && (fl & F_PRUNE_BL);
    for (uint64_t q = s->lo; q < s->hi; ++q) {
        uint32_t u = s->qu[q], v = s->qv[q];
        uint8_t code;
        if (u >= n || v >= n) { s->err = ORC_E_RANGE; break; }
        const uint64_t *dlo_u = s->dl_out + (uint64_t)u * wdl, *dli_u = s->dl_in + (uint64_t)u * wdl;
        const uint64_t *dlo_v = s->dl_out + (uint64_t)v * wdl, *dli_v = s->dl_in + (uint64_t)v * wdl;
        const uint64_t *bli_u = s->bl_in + (uint64_t)u * wbl, *blo_u = s->bl_out + (uint64_t)u * wbl;
        const uint64_t *bli_v = s->bl_in + (uint64_t)v * wbl, *blo_v = s->bl_out + (uint64_t)v * wbl;
        if (u == v) code = A_REFLEXIVE;
        else if (use_dl && and_nz(dlo_u, dli_v, wdl)) code = A_DL_POS;
        else if (use_bl && (andnot_nz(bli_u, bli_v, wbl) || andnot_nz(blo_v, blo_u, wbl))) code = A_BL_NEG;
        else if (use_dl && (fl & F_THM1) && and_nz(dlo_v, dli_u, wdl)) code = A_THM1;
        else if (use_dl && (fl & F_THM2) && (and_nz(dlo_u, dli_u, wdl) || and_nz(dlo_v, dli_v, wdl))) code = A_THM2;
        else {
            if (++epoch == 0) { memset(stamp, 0, (size_t)n * 4); epoch = 1; }
            stamp[u] = epoch;
            uint32_t head = 0, tail = 0;
            queue[tail++] = u;
            code = A_BFS_NEG;
            while (head < tail && code == A_BFS_NEG) {
                uint32_t w = queue[head++];
                for (uint64_t e = s->ptr[w]; e < s->ptr[w + 1]; ++e) {
                    uint32_t x = s->col[e];
                    if (x == v) { code = A_BFS_POS; break; }
                    if (stamp[x] == epoch) continue;
                    stamp[x] = epoch;
                    if (prune_dl && and_nz(dlo_u, s->dl_in + (uint64_t)x * wdl, wdl)) continue;
                    if (prune_bl && (andnot_nz(s->bl_in + (uint64_t)x * wbl, bli_v, wbl) ||
                                     andnot_nz(blo_v, s->bl_out + (uint64_t)x * wbl, wbl)))
                        continue;
                    queue[tail++] = x;
                }
            }
        }
        s->codes[q] = code;
    }
    free(stamp);
    free(queue);
    return NULL;
}

int orc_csr_query_batch(uint32_t n, const uint64_t *ptr, const uint32_t *col, uint32_t k, uint32_t k_prime,
                        const uint64_t *dl_in, const uint64_t *dl_out, const uint64_t *bl_in,
                        const uint64_t *bl_out, const uint32_t *qu, const uint32_t *qv, uint64_t q,
                        uint32_t flags, uint8_t *codes, int threads) {
    uint32_t wdl = (k + 63) / 64, wbl = (k_prime + 63) / 64;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads * 2 > q) threads = 1;
    cslice *sl = (cslice *)calloc(threads, sizeof(cslice));
    uint64_t chunk = (q + threads - 1) / threads;
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; ++i) {
        uint64_t lo = (uint64_t)i * chunk, hi = lo + chunk;
        if (lo > q) lo = q;
        if (hi > q) hi = q;
        cslice t = {n, wdl, wbl, ptr, col, dl_in, dl_out, bl_in, bl_out, qu, qv, codes, flags, lo, hi, 0};
        sl[i] = t;
        pthread_create(&tid[i], NULL, csr_query_slice, &sl[i]);
    }
    int err = 0;
    for (int i = 0; i < threads; ++i) { pthread_join(tid[i], NULL); if (sl[i].err) err = sl[i].err; }
    free(tid);
    free(sl);
    return err;
}
