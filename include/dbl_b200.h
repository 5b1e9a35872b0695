/*
 * dbl_b200.h -- C ABI of the B200-native DBL reachability engine.
 *
 * The reference (dblreach, pure Python) has no FFI; its boundary is the
 * Python API listed in SURVEY.md §8(b).  Each entry point below replaces
 * one reference function (paths relative to
 * /root/reference/pkg/src/dblreach/).  The Python shim
 * paper_2101_09441_b200/ (_native.py binds these with ctypes; graph.py,
 * labels.py, queries.py, updates.py keep the reference's own names) is the
 * drop-in; INTEGRATION.md shows the binding a reference maintainer adds.
 *
 * Conventions
 *  - Every call returns a dbl_status; DBL_OK == 0.  On failure
 *    dbl_last_error() returns a thread-local message.  Status codes map 1:1
 *    onto the reference's DblError subclasses (errors.py:4-40).
 *  - Vertex ids are uint32; vertex count n < 2^32; edge count < 2^32.
 *  - Pointer arguments marked (host|device) honour `mem`: DBL_MEM_HOST means
 *    pageable/pinned host memory (the call stages copies itself),
 *    DBL_MEM_DEVICE means device memory on the handle's GPU.  Device inputs
 *    are read only after the work already queued on the legacy default
 *    stream (the handle's own stream waits on it through an event, without
 *    a host sync); a caller producing them on another stream synchronises
 *    that stream first.
 *  - Handles own all device state (including per-call workspaces), so a
 *    graph handle serves one host thread at a time; its calls are
 *    serialised on the handle's stream.  For concurrent queries use one
 *    replica per thread or dbl_query_multi.  Queries are read-only and may
 *    not overlap an insertion (reference contract: pkg/README.md:179-183).
 *  - Label bit i lives in bit (i % 64) of word (i / 64), least-significant
 *    word first (pkg/docs/snapshot-format.md:38-42).
 */
#ifndef DBL_B200_H
#define DBL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DBL_OK = 0,
    DBL_E_VERTEX_RANGE = 1,   /* VertexRangeError      errors.py:8-9   */
    DBL_E_CONFIG = 2,         /* ConfigError           errors.py:23-24 */
    DBL_E_MISMATCH = 3,       /* IndexGraphMismatchError errors.py:27-28 */
    DBL_E_CUDA = 4,           /* device failure (no reference analogue) */
    DBL_E_ARG = 5,            /* bad pointer / size (TypeError analogue) */
    DBL_E_OOM = 6             /* device allocation failed */
} dbl_status;

typedef enum { DBL_MEM_HOST = 0, DBL_MEM_DEVICE = 1 } dbl_mem;

/* LandmarkStrategy, labels.py:31-46 */
typedef enum { DBL_STRAT_MAX = 0, DBL_STRAT_MIN = 1, DBL_STRAT_SUM = 2,
               DBL_STRAT_PRODUCT = 3 } dbl_strategy;

/* QueryFlags, queries.py:59-75 (bit set; DBL_FLAGS_DEFAULT = all on) */
#define DBL_F_USE_DL   1u
#define DBL_F_USE_BL   2u
#define DBL_F_THM1     4u
#define DBL_F_THM2     8u
#define DBL_F_PRUNE_DL 16u
#define DBL_F_PRUNE_BL 32u
#define DBL_FLAGS_DEFAULT 63u

/* AnsweredBy codes in _ANSWER_ORDER, queries.py:40-47, 188-189.
 * reachable == (code == REFLEXIVE || DL_POSITIVE || BFS_POSITIVE). */
enum { DBL_REFLEXIVE = 0, DBL_DL_POSITIVE = 1, DBL_BL_NEGATIVE = 2,
       DBL_THM1_NEGATIVE = 3, DBL_THM2_NEGATIVE = 4, DBL_BFS_POSITIVE = 5,
       DBL_BFS_NEGATIVE = 6 };

typedef struct dbl_graph dbl_graph;
typedef struct dbl_index dbl_index;

/* IndexConfig, labels.py:92-116 */
typedef struct {
    uint32_t k;               /* landmark bits, 0 <= k <= n        */
    uint32_t k_prime;         /* leaf-hash buckets, >= 1           */
    int32_t strategy;         /* dbl_strategy                      */
    uint64_t leaf_threshold;  /* r                                 */
    uint64_t hash_seed;
} dbl_config;

/* UpdateStats, updates.py:31-50 (single-edge insert: exact) */
typedef struct {
    uint32_t visited;
    uint32_t labels_changed;
    uint32_t early_terminated;
    uint32_t inserted;        /* 1 if the edge was new (add_edge's return) */
} dbl_update_stats;

/* Batched insertion statistics (no reference analogue: the reference only
 * inserts one edge at a time; see DESIGN.md for how these relate). */
typedef struct {
    uint64_t requested;       /* edges passed in                           */
    uint64_t inserted;        /* new distinct edges added to the graph     */
    uint64_t certified;       /* edges whose pre-batch DL labels certified u->v */
    uint64_t labels_changed;  /* distinct (vertex, direction) label changes */
    uint32_t levels;          /* fixpoint levels run                       */
    uint32_t delta_merged;    /* 1 if the delta adjacency was compacted    */
    uint64_t fix_items;       /* delta fixpoint: frontier items expanded   */
    uint64_t fix_edges;       /* delta fixpoint: edges relaxed             */
} dbl_batch_stats;

/* ---------------------------------------------------------------- misc */
const char *dbl_last_error(void);
int dbl_version(void);
/* number of kernels this process launched through the library */
uint64_t dbl_kernel_launches(void);
/* Return the library's cached device blocks to the driver (cudaFree). */
dbl_status dbl_release_cached_memory(void);
/* leaf_hash, labels.py:119-137, evaluated on the device for a batch */
dbl_status dbl_leaf_hash(const uint64_t *ids, uint64_t count, uint32_t k_prime,
                         uint64_t seed, uint32_t *out_buckets, int device);

/* --------------------------------------------------------------- graph */
/* DynamicGraph + add_edge dedup (graph.py:31-66): builds CSR (forward) and
 * CSC (reverse) on `device` from an edge list; duplicate edges collapse,
 * self-loops are kept (they count toward degrees as in the reference). */
dbl_status dbl_graph_create(uint32_t n, const uint32_t *src, const uint32_t *dst,
                            uint64_t m, dbl_mem mem, int device, dbl_graph **out);
dbl_status dbl_graph_free(dbl_graph *g);
/* vertex_count / edge_count (graph.py:44-46) */
dbl_status dbl_graph_info(const dbl_graph *g, uint32_t *n, uint64_t *m);
/* in_degree / out_degree for all vertices (graph.py:93-99), host out */
dbl_status dbl_graph_degrees(const dbl_graph *g, uint32_t *indeg, uint32_t *outdeg);
/* has_edge (graph.py:80-81) for a batch of pairs, host in/out */
dbl_status dbl_graph_has_edges(const dbl_graph *g, const uint32_t *u, const uint32_t *v,
                               uint64_t count, uint8_t *out);
/* edges() (graph.py:101-105): all edges sorted by (src, dst), host out;
 * arrays must hold dbl_graph_info's m entries. */
dbl_status dbl_graph_edges(const dbl_graph *g, uint32_t *src, uint32_t *dst);
/* One direction's adjacency (reverse = 0: out-edges, 1: in-edges) as plain
 * CSR, host out: ptr[n+1] and col[m] (rows: base edges then inserted ones). */
dbl_status dbl_graph_adjacency(const dbl_graph *g, int reverse, uint32_t *ptr, uint32_t *col);
/* add_edge (graph.py:56-66) for a batch, graph only (no label upkeep):
 * duplicates collapse; *out_inserted = number of new distinct edges. */
dbl_status dbl_graph_add_edges(dbl_graph *g, const uint32_t *u, const uint32_t *v,
                               uint64_t count, uint64_t *out_inserted);
/* add_vertex (graph.py:48-51) x count; ids n..n+count-1 get no edges */
dbl_status dbl_graph_add_vertices(dbl_graph *g, uint32_t count);

/* ------------------------------------------------------------ metadata */
/* select_landmarks, labels.py:140-147: top-k by (-score, id), host out */
dbl_status dbl_select_landmarks(const dbl_graph *g, uint32_t k, int32_t strategy,
                                uint32_t *out_ids);
/* select_leaves, labels.py:150-181.  Optional bucket override
 * (ovr_ids/ovr_buckets, n_ovr entries, host).  Outputs (host, length n):
 * flags bit0 = leaves_in, bit1 = leaves_out; bucket valid where flags!=0. */
dbl_status dbl_select_leaves(const dbl_graph *g, uint64_t threshold, uint32_t k_prime,
                             uint64_t hash_seed, const uint32_t *ovr_ids,
                             const uint32_t *ovr_buckets, uint32_t n_ovr,
                             uint8_t *out_flags, uint32_t *out_bucket);

/* --------------------------------------------------------------- index */
/* build_index, labels.py:263-306.  landmarks (host, k ids) pins the
 * landmark order, else select_landmarks runs on the device.  leaf_flags +
 * bucket (host, n each) pin the leaf metadata (the rebuild_index path,
 * labels.py:309-312), else select_leaves runs on the device with the
 * optional override table. */
dbl_status dbl_index_build(const dbl_graph *g, const dbl_config *cfg,
                           const uint32_t *landmarks, const uint8_t *leaf_flags,
                           const uint32_t *bucket, const uint32_t *ovr_ids,
                           const uint32_t *ovr_buckets, uint32_t n_ovr,
                           dbl_index **out);
/* Metadata selection (or pinning, as dbl_index_build) and label seeding
 * only -- no propagation; pair with dbl_index_build_words for sharded
 * builds. */
dbl_status dbl_index_create(const dbl_graph *g, const dbl_config *cfg,
                            const uint32_t *landmarks, const uint8_t *leaf_flags,
                            const uint32_t *bucket, const uint32_t *ovr_ids,
                            const uint32_t *ovr_buckets, uint32_t n_ovr,
                            dbl_index **out);
/* rebuild_index, labels.py:309-312: fresh build into `idx` reusing its
 * frozen metadata on the current graph. */
dbl_status dbl_index_rebuild(const dbl_graph *g, dbl_index *idx);
dbl_status dbl_index_free(dbl_index *idx);
dbl_status dbl_index_info(const dbl_index *idx, uint32_t *n, dbl_config *cfg);
/* Frozen metadata (host out): landmarks[k], leaf flags[n], bucket[n]. */
dbl_status dbl_index_metadata(const dbl_index *idx, uint32_t *landmarks,
                              uint8_t *leaf_flags, uint32_t *bucket);
/* Labels as u64 words, LSW first (host out).  dl_* hold n*ceil(k/64)
 * words, bl_* n*ceil(k'/64); any pointer may be NULL. */
dbl_status dbl_index_export(const dbl_index *idx, uint64_t *dl_in, uint64_t *dl_out,
                            uint64_t *bl_in, uint64_t *bl_out);
/* Load labels (host in) into an index (snapshot import). */
dbl_status dbl_index_import(dbl_index *idx, const uint64_t *dl_in, const uint64_t *dl_out,
                            const uint64_t *bl_in, const uint64_t *bl_out);
/* labels_equal (labels.py:238-244), evaluated on the device */
dbl_status dbl_index_equal(const dbl_index *a, const dbl_index *b, int *out_equal);
/* grow_to (labels.py:209-216): new vertices get empty labels */
dbl_status dbl_index_grow(dbl_index *idx, uint32_t n);
/* dl_intersec (labels.py:315-319) and bl_contain (labels.py:322-327) for
 * a batch of (x, y) pairs evaluated on the device; host in/out. */
dbl_status dbl_label_tests(const dbl_index *idx, const uint32_t *x, const uint32_t *y,
                           uint64_t count, uint8_t *out_dl_intersec, uint8_t *out_bl_contain);
/* Device pointer to the AoS record table and its record stride in words:
 * record v starts at word v * stride and holds dl_in|bl_in|dl_out|bl_out
 * (2*(ceil(k/64)+ceil(k'/64)) words; records wider than 32 bytes are padded
 * to 64 or a multiple of 128 bytes, pad words unspecified), for zero-copy
 * consumers.  Read-only: the index keeps derived state (the query digest)
 * that only its own entry points keep in step with the records. */
dbl_status dbl_index_records(const dbl_index *idx, uint64_t **dev_records,
                             uint32_t *words_per_record);

/* Query digest (no reference counterpart: derived state of this engine):
 * out[x] (n u32, host) summarises x's labels -- bit 0/1: dl_out has
 * landmark 0 / any other landmark, bit 2/3: the same for dl_in, bits 4..17 /
 * 18..31: bl_in / bl_out with bucket b folded onto bit (b % 64) % 14.  Query
 * batches decide a pair from the two digests when they prove rule 1 or rule
 * 2 of queries.py:102-108 and read the records otherwise.  Builds compute
 * it; inserts keep a current digest current (single inserts OR the new
 * label bits' digest bits in, batches recompute the changed vertices); other
 * label writes leave it stale until a batch of >= 64k pairs or this call
 * recomputes it.  *was_current (optional) tells whether it was current. */
dbl_status dbl_index_digest(const dbl_index *idx, const dbl_graph *g, uint32_t *out, int *was_current);

/* -------------------------------------------------------------- queries */
/* query_batch, queries.py:94-142, 210-249: label rules 0..4 on every
 * pair, then the batched pruned BFS for the rest.  codes[i] is the
 * AnsweredBy code; visited[i] (optional) is 0 iff label-answered.
 * Raises DBL_E_VERTEX_RANGE if any id >= n, DBL_E_MISMATCH if the graph and
 * index vertex counts differ (queries.py:88-91). */
dbl_status dbl_query(const dbl_index *idx, const dbl_graph *g, const uint32_t *u,
                     const uint32_t *v, uint64_t count, uint32_t flags, uint8_t *codes,
                     uint32_t *visited, dbl_mem mem);
/* query, queries.py:94-142, for one pair with scalar arguments (the
 * per-call path: a resident service answers it without a kernel launch,
 * see DESIGN.md §4): out[0] = AnsweredBy code, out[1] = visited. */
dbl_status dbl_query_one(const dbl_index *idx, const dbl_graph *g, uint32_t u, uint32_t v, uint32_t flags,
                         uint32_t *out);
/* Same as dbl_query but enqueued on the handle's stream without a final
 * synchronisation (device memory only); dbl_sync waits for it.  Unlike the
 * synchronous calls it does not order itself after the legacy default
 * stream: produce u / v on the handle's stream (dbl_stream) or synchronise
 * their producer first.  A batch
 * whose pruned BFS outgrows the shared-memory tables needs the dense
 * workspace (n x 32 bytes per CTA), which is allocated on first need: such a
 * batch is completed by dbl_sync (it re-runs the batch), so call dbl_sync
 * before reading the codes of an async batch. */
dbl_status dbl_query_async(const dbl_index *idx, const dbl_graph *g, const uint32_t *u,
                           const uint32_t *v, uint64_t count, uint32_t flags,
                           uint8_t *codes, uint32_t *visited);
dbl_status dbl_sync(const dbl_graph *g);
/* query_batch over several devices (the reference's worker
 * pool, queries.py:224-247): the host batch is cut into ndev contiguous
 * slices of ceil(count / ndev) pairs (queries.py:231-232) and slice d is
 * answered by (idx[d], g[d]) -- identical replicas, one per device -- on its
 * own host thread, all slices concurrently.  Results land in input order.
 * DBL_MEM_HOST: pinned or pageable host buffers.  DBL_MEM_DEVICE: u, v,
 * codes (and visited) all on one GPU; the other devices access them by peer
 * access over NVLink (enabled here; the producer of u / v must be finished).
 * Each graph handle may appear once.  Errors name the failing slice. */
dbl_status dbl_query_multi(const dbl_index *const *idx, const dbl_graph *const *g, uint32_t ndev,
                           const uint32_t *u, const uint32_t *v, uint64_t count, uint32_t flags,
                           uint8_t *codes, uint32_t *visited, dbl_mem mem);
/* Counters of the last query batch (8 x u32): [0] queries finished by the
 * 64-query group kernel, [1] range-error flag, [3] groups re-run densely. */
dbl_status dbl_query_counters(const dbl_graph *g, uint32_t *out8);
/* The CUDA stream all work of `g` (and indexes built on it) runs on. */
dbl_status dbl_stream(const dbl_graph *g, void **cuda_stream);

/* ------------------------------------------------------------- updates */
/* insert_edge, updates.py:112-137, exact UpdateStats. */
dbl_status dbl_insert_edge(dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v,
                           dbl_update_stats *stats);
/* A batch of insertions; labels end equal to the sequential insert_edge
 * loop and to rebuild_index (least fixpoint). */
dbl_status dbl_insert_edges(dbl_index *idx, dbl_graph *g, const uint32_t *u,
                            const uint32_t *v, uint64_t count, dbl_mem mem,
                            dbl_batch_stats *stats);

/* ------------------------------------------------ multi-GPU word shards */
/* Rebuild only the listed record words (indices into the AoS record, see
 * dbl_index_records) from the index's frozen metadata.  Word families are
 * independent fixpoints, so GPUs can split them. */
dbl_status dbl_index_build_words(const dbl_graph *g, dbl_index *idx, const uint32_t *words,
                                 uint32_t nwords);
/* Gather record words into a word-major device slab (nw x n u64) on
 * `cuda_stream`, and the inverse scatter (the record interleave that follows
 * the NCCL allgather). */
dbl_status dbl_index_pack_words(const dbl_index *idx, const uint32_t *words, uint32_t nw,
                                uint64_t *dev_slab, void *cuda_stream);
dbl_status dbl_index_unpack_words(dbl_index *idx, const uint32_t *words, uint32_t nw,
                                  const uint64_t *dev_slab, void *cuda_stream);

/* ------------------------------------------------------------ verifier */
/* verify_labels (updates.py:323-363) on the device: the union-fixpoint
 * check over every (vertex, half) and, if `exhaustive`, a diff against a
 * fresh rebuild from the frozen metadata.  Writes up to max_out violation
 * rows (vertex, half 0 = in / 1 = out, expected and actual half words,
 * ceil(k/64)+ceil(k'/64) each, dl words first); *out_count = total found. */
dbl_status dbl_verify(const dbl_index *idx, const dbl_graph *g, int exhaustive, uint64_t max_out,
                      uint64_t *out_count, uint32_t *out_vertex, uint8_t *out_half,
                      uint64_t *out_expected, uint64_t *out_actual);

/* ----------------------------------------------------- synthetic inputs */
/* Counter-based R-MAT generator (configs 3-5): m edges over 2^scale
 * vertices with quadrant probabilities a, b, c (d = 1-a-b-c) into device
 * buffers; self-loops are kept (callers drop them). Deterministic in seed. */
dbl_status dbl_rmat_generate(uint32_t scale, uint64_t m, uint64_t seed, double a, double b, double c,
                             uint32_t *dev_src, uint32_t *dev_dst, int device);

/* ------------------------------------------------------ instrumentation */
/* Level-synchronous (Jacobi) work model of SURVEY.md §8(d) for every
 * 64-bit word family of `idx`'s metadata on `g`: per family f (order:
 * dl_in words, bl_in words, dl_out words, bl_out words) V_f, E_f and the
 * level count.  Arrays hold 2*(ceil(k/64)+ceil(k'/64)) entries. */
dbl_status dbl_work_model(const dbl_index *idx, const dbl_graph *g, uint64_t *V,
                          uint64_t *E, uint32_t *levels);
/* Executed work of the last build on `g` (the bench's build roofline counts
 * the bytes of this work, not the level-synchronous model above). */
typedef struct {
    uint64_t n, m;               /* graph size at the build                          */
    uint32_t record_bytes;       /* record stride in bytes                           */
    uint32_t flags;              /* bit0 prep wrote the seeded records; bit1 the pivot
                                    pass wrote every record whole; bit2 the pivot pass
                                    ORed its unions into the records (read + write);
                                    bit3 the pivot sweeps hit their cap; bit4 word build */
    uint32_t sweeps, steps;      /* pivot reach: bottom-up sweeps, all steps         */
    uint32_t fix_levels, fix_runs; /* label fixpoint: levels over all runs, runs     */
    uint64_t bu_tests;           /* pivot bottom-up (vertex, direction) tests        */
    uint64_t bu_probes;          /* their neighbour probes                           */
    uint64_t td_vertices, td_edges; /* pivot top-down levels                        */
    uint64_t union_records;      /* records the pivot's union pass touched           */
    uint64_t fix_items, fix_edges;  /* label fixpoint: frontier items, relaxed edges
                                       (first 32 levels of each run)                 */
} dbl_build_work;
dbl_status dbl_build_work_stats(const dbl_graph *g, dbl_build_work *out);
/* on != 0: later builds on g run the instrumented pivot kernel, which also
 * fills the pivot fields of the dbl_build_work struct (the product kernel
 * carries no counters, so without instrumentation those fields stay 0), and
 * query batches record CUDA events around their kernels for
 * dbl_last_timings (two extra event records per batch on the stream). */
dbl_status dbl_graph_instrument(dbl_graph *g, int on);
/* Device time (ms) of the last fixpoint launch and (instrumented graphs
 * only, else 0) of the last query batch's kernels, measured with CUDA
 * events on the handle's stream. */
dbl_status dbl_last_timings(const dbl_graph *g, float *fixpoint_ms, float *label_ms,
                            float *bfs_ms);

#ifdef __cplusplus
}
#endif
#endif
