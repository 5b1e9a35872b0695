// internal.cuh -- shared device structures of the DBL engine (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>
#include <atomic>
#include <map>
#include <string>
#include <tuple>

#include "dbl_b200.h"

// Compile-time switches.  Kernel-variant experiments are chosen by -D flags
// in build.build_variant builds, never by the environment of a product run.
#ifndef DBL_TRACE
#define DBL_TRACE 0          // 1: host-side phase times to stderr (debug builds)
#endif
// Checked build (build.build_variant("checked", ["DBL_CHECKED=1"])): device
// bounds checks on every adjacency column id, queue slot and record index
// the kernels derive from data; a failure prints the site and traps, so the
// next CUDA call of the test fails.  The substitute for compute-sanitizer
// memcheck, which this pool does not run.
#ifndef DBL_CHECKED
#define DBL_CHECKED 0
#endif
#if DBL_CHECKED
#include <cstdio>
#define DBL_DCHECK(c)                                                                     \
    do {                                                                                  \
        if (!(c)) {                                                                       \
            printf("DBL_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);              \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define DBL_DCHECK(c) ((void)0)
#endif

namespace dbl {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t DELTA_BIT = 0x80000000u;
#ifndef DBL_FIX_THREADS
#define DBL_FIX_THREADS 256
#endif
constexpr int FIX_THREADS = DBL_FIX_THREADS;
constexpr int MAX_GROUP_WORDS = 8;        // words propagated together by one fixpoint
constexpr int MAX_SHARD_WORDS = 32;  // words per record half (2 halves <= 64-bit word mask)

// ---------------------------------------------------------------- errors --
void set_error(const std::string &msg);
dbl_status cuda_fail(cudaError_t e, const char *what);
std::atomic<uint64_t> &launch_counter();
// blocks per SM of `fn` (dynamic smem opted in), cached per device
dbl_status kernel_occupancy(const void *fn, int threads, size_t smem, int *bps);

#define DBL_CUDA(call)                                                         \
    do {                                                                       \
        cudaError_t _e = (call);                                               \
        if (_e != cudaSuccess) return ::dbl::cuda_fail(_e, #call);             \
    } while (0)
#define DBL_LAUNCHED() (++::dbl::launch_counter())
#define DBL_CHECK_LAUNCH(what)                                                 \
    do {                                                                       \
        DBL_LAUNCHED();                                                        \
        cudaError_t _e = cudaGetLastError();                                   \
        if (_e != cudaSuccess) return ::dbl::cuda_fail(_e, what);              \
    } while (0)

// Caching device allocator (abi.cu): size classes of 1/8 octave, blocks are
// recycled instead of cudaFree'd, so per-call workspaces cost no
// cudaMalloc/cudaFree synchronisation after warm-up.
cudaError_t pool_alloc(void **p, size_t *bytes, int *device);
void pool_free(void *p, size_t bytes, int device);
void pool_trim();
void set_stream(cudaStream_t s);  // stream that subsequent pool traffic belongs to
void set_stream_synced();         // the device was just synchronised: frees are reusable without waiting
// Device-memory inputs are produced by the caller on the legacy default
// stream (torch's, unless the caller set another and synchronised it); the
// engine's stream is non-blocking, so it waits for that stream's pending work
// through an event (no host sync) before reading them.
dbl_status order_after_caller(dbl_graph *g);
void pool_forget_stream(cudaStream_t s);  // before a stream is destroyed
// Debug phase timer: a -DDBL_TRACE=1 build prints host-side phase times to stderr.
void trace(const char *what, cudaStream_t s);

// grow-only device buffer backed by the caching allocator
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    int dev = 0;
    dbl_status ensure(size_t need) {
        if (need <= bytes) return DBL_OK;
        release();
        size_t nb = need < 256 ? 256 : need;
        cudaError_t e = pool_alloc(&p, &nb, &dev);
        if (e != cudaSuccess) { cudaGetLastError(); p = nullptr; return cuda_fail(e, "cudaMalloc(workspace)"); }
        bytes = nb;
        return DBL_OK;
    }
    // grow by at least 1.5x so arrays that creep upward (delta adjacency)
    // are not reallocated on every call
    dbl_status ensure_geometric(size_t need) {
        if (need <= bytes) return DBL_OK;
        const size_t grown = bytes + bytes / 2;
        return ensure(need > grown ? need : grown);
    }
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
    void release() { if (p) pool_free(p, bytes, dev); p = nullptr; bytes = 0; }
};

// Pinned host staging buffer (grow-only).
struct HostBuf {
    void *p = nullptr;
    size_t bytes = 0;
    dbl_status ensure(size_t need) {
        if (need <= bytes) return DBL_OK;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMallocHost(&p, need);
        if (e != cudaSuccess) { cudaGetLastError(); return cuda_fail(e, "cudaMallocHost"); }
        bytes = need;
        return DBL_OK;
    }
    void release() { if (p) cudaFreeHost(p); p = nullptr; bytes = 0; }
};

// One traversal direction's adjacency: base CSR + delta CSR (insertions).
struct Adj {
    const uint32_t *ptr;    // n+1
    const uint32_t *col;
    const uint32_t *dptr;   // n+1 or nullptr
    const uint32_t *dcol;
    uint32_t n;             // vertex count (bounds of every column id; DBL_DCHECK)
    uint32_t pad;
};

// Executed work of the last build on a graph (dbl_build_work_stats).
struct BuildWork {
    uint64_t fix_items = 0, fix_edges = 0;
    uint32_t fix_levels = 0, fix_runs = 0;
    uint32_t flags = 0;   // see dbl_build_work in dbl_b200.h
    uint32_t rs = 0;      // record stride (words)
};

// Arguments of one query batch (kept by the graph for dbl_sync).
struct QueryArgs {
    const dbl_index *idx;
    const uint32_t *u, *v;
    uint8_t *codes;
    uint32_t *visited;
    uint64_t count;
    uint32_t flags;
};

// Frontier work items: one per nonempty adjacency segment of a frontier
// vertex: (vertex, first edge, length | DELTA_BIT, offset of its first edge
// in the level's edge space).  eoff is monotone in the item index, so warps
// can split a level into equal edge ranges and binary-search their items.
struct Queue {
    uint32_t *x;
    uint32_t *start;
    uint32_t *len;
    uint32_t *eoff;
};

// Device state of the fused build prep (select.cu): score histogram for the
// landmark top-k, candidate counts, and the flags the host reads once the
// build has finished (no host round trip inside the build).
#ifndef DBL_PREP_CAND_CAP
#define DBL_PREP_CAND_CAP 8192
#endif
constexpr uint32_t PREP_CAND_CAP = DBL_PREP_CAND_CAP;   // top-k candidates sorted on chip
struct PrepState {
    uint32_t hist[65];
    uint32_t n_above, n_tie;
    uint32_t fallback;           // candidates exceeded PREP_CAND_CAP: host re-selects
    unsigned long long err;      // bucket override outside [0, k')
};

// Device control block of one fixpoint run.
struct Ctrl {
    unsigned long long cnt[2][2];   // (items << 32 | edges) per [level % 2][direction]
    uint32_t ticket[2];              // relax-phase edge tickets per level % 2
    uint32_t levels;
    uint32_t overflow;
    uint32_t seed_changed[2];
    uint32_t pad;
    unsigned long long changed[2];   // distinct vertices whose label grew
    unsigned long long error;        // range errors etc.
    unsigned long long level_edges[32];  // edges expanded per level (first 32 levels, both directions)
    unsigned long long level_items[32];
    unsigned long long level_t[64];       // globaltimer at each phase boundary (block 0)
    unsigned long long dbg[4];            // trace builds: level-0 compaction per warp (max, sum, min, start spread)
};

// One direction of a fixpoint: label words [lab + v*stride, +nw) propagate
// along `adj` (forward CSR for in-labels, reverse CSC for out-labels).
struct DirParams {
    Adj adj;                  // push adjacency (forward for in-labels)
    Adj padj;                 // pull adjacency (the opposite direction)
    uint64_t *lab;
    uint32_t stride;
    int al;                   // lab's word offset in a 32-byte chunk (stride % 4 == 0), else -1
    uint32_t *bits;           // next-frontier bitmap (n bits)
    uint32_t *cur;            // current-frontier bitmap (pull levels)
    Queue q;                  // current level's work items
    uint32_t cap;
    uint32_t *changed_bits;   // nullptr unless counting distinct changes
};

struct FixParams {
    DirParams d[2];
    Ctrl *ctrl;
    uint64_t m_base, m_delta;
    uint32_t pull_div;        // a direction pulls when its frontier edges exceed m / pull_div
    uint32_t n;
    uint32_t active;          // bit d: direction d has words in this run
    uint32_t max_levels;
};

}  // namespace dbl

// ------------------------------------------------------------- handles --
struct dbl_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint32_t n = 0;
    uint64_t m_base = 0, m_delta = 0;
    // base adjacency
    dbl::DevBuf fptr, fcol, rptr, rcol;
    // delta adjacency (insertions since the last compaction)
    dbl::DevBuf dfptr, dfcol, drptr, drcol, dkeys_f, dkeys_r, dmerge;
    // traversal workspace shared by builds/inserts on this graph
    dbl::DevBuf stamp[2];     // per-direction frontier bitmaps
    dbl::DevBuf qbuf[2][2];   // [direction][0] work-item queue storage
    uint32_t qcap = 0;
    dbl::DevBuf ctrl;
    dbl::DevBuf haspred;      // build: per direction, vertices with predecessors (prep -> pivot sweeps)
    dbl::DevBuf reach;        // pivot reachability: n x {from pivot, to pivot} u64 + 2 bitmaps + unions
    unsigned long long *reach_work = nullptr;   // the last pivot pass's work counters (in `reach`)
    unsigned int *reach_chg = nullptr;          // its step words: [3] capped, [4] steps, [5] sweeps
    dbl::BuildWork last_build{}, last_insert{};
    bool instrument = false;                    // builds count their executed work (dbl_graph_instrument)
    // single-edge inserts not yet folded into the delta adjacency
    // (insert_one.cu; graph_flush_pending folds them before any other use)
    dbl::DevBuf pend, pend_sort;
    uint32_t n_pend = 0;
    dbl::HostBuf one_out;
    dbl::DevBuf changed_bits;
    // generic scratch
    dbl::DevBuf cub_tmp, scratch_a, scratch_b, scratch_c, scratch_d;
    dbl::DevBuf ins_in, ins_keys, ins_alt, ins_newk, ins_err;   // insert-batch workspaces
    std::map<std::tuple<int, uint64_t, uint64_t>, size_t> cub_sizes;   // cub_cached
    // the insert batch's radix sort replayed as a captured CUDA graph
    // (graph.cu sort_keys_replay): key = buffers, size, bits, temporary storage
    cudaGraphExec_t sort_exec = nullptr;
    std::tuple<const void *, const void *, uint64_t, int, const void *> sort_key{}, sort_seen{};
    uint64_t *sort_out = nullptr;
    bool sort_graph_off = false;
    dbl::DevBuf prep;                     // PrepState + top-k candidates
    dbl::HostBuf host_stage;
    dbl::HostBuf q_host_res;              // pinned result words of the last query batch
    dbl::HostBuf q_stage;                 // pinned staging of small pageable query batches
    // query workspace
    dbl::DevBuf q_in, q_codes, q_vis, q_pending, q_counters, q_dense, q_errs;
    cudaStream_t cstream[2] = {nullptr, nullptr};   // H2D / D2H copy streams
    cudaEvent_t cev[33] = {};
    uint64_t q_pending_cap = 0;
    dbl::QueryArgs q_last{};              // arguments of the last batch (dbl_sync re-runs it if it needed the dense workspace)
    bool q_timed_bfs = false;            // last batch ran the separate BFS kernels (ev[3] -> ev[4])
    uint64_t topo_version = 0;           // bumped whenever adjacency buffers change
    int sm_count = 148;
    int coop_blocks = 0;      // co-resident blocks for the fixpoint kernel
    cudaEvent_t ev[6] = {};
    cudaEvent_t ev_in = nullptr;   // orders the engine stream after the caller's (order_after_caller)
    float t_fix = 0, t_label = 0, t_bfs = 0;
    // per-call query service (query.cu): one resident warp answering single
    // query() calls through a mailbox in pinned host memory
    cudaStream_t sstream = nullptr;
    dbl::HostBuf sbox;
    const dbl_index *s_idx = nullptr;   // index the running service reads
    uint64_t s_ver = 0;                 // its label version at launch
    uint32_t s_seq = 0;                 // last request number posted
    bool s_running = false;
    bool s_dig = false;                 // the service keeps the digest current (it was at launch)
};

// Record stride (u64 words) for half-width H = wdl + wbl.  L2 fills whole
// 128-byte lines on the random misses of the query gather, so a record never
// straddles a line: 16- and 32-byte records stay packed, wider ones are padded
// to 64 or a multiple of 128 bytes (cfg5, k = 256: 80 -> 128 bytes, 1.5 -> 1
// lines per endpoint).  The out-half starts at word H as before.
__host__ __device__ constexpr uint32_t rec_stride(uint32_t H) {
    return 2 * H <= 4 ? 2 * H : (2 * H <= 8 ? 8u : ((2 * H + 15) & ~15u));
}

struct dbl_index {
    int device = 0;
    uint32_t n = 0;
    dbl_config cfg{};
    uint32_t wdl = 0, wbl = 0, rw = 0;  // words: dl, bl, per record (2H)
    uint32_t rs = 0;                     // record stride in words (rec_stride(H) >= rw; pad words unspecified)
    dbl::DevBuf rec;                     // n * rs u64
    dbl::DevBuf landmarks;               // k u32
    dbl::DevBuf leaf_flags;              // n u8
    dbl::DevBuf bucket;                  // n u32
    // metadata still to be selected by the build's fused prep pass
    // (dbl_index_build): landmarks, leaves (with an optional override table)
    bool sel_landmarks = false, sel_leaves = false;
    dbl::DevBuf ovr;                     // n u32 override buckets (0xffffffff = none)
    // pivot sets kept for query pruning (written by the build's reach kernel):
    // dmask = vertices reached from the pivot h (a subset of D(h)),
    // sccmask = DL bits of the landmarks in h's SCC.  A query whose dl_out[u]
    // meets sccmask prunes every x in D(h) (queries.py:137-138) on one bit.
    dbl::DevBuf dmask, sccmask;
    uint32_t dmask_n = 0;                // vertices covered by dmask
    bool has_scc = false;
    // Label digest (query.cu): one u32 per vertex summarising its four label
    // families, n x 4 bytes, so a query batch decides most pairs from an
    // L2-resident table and reads the full records only for the rest.
    // `version` moves on every label change (each ABI entry that writes
    // records); the digest is current iff digest_version == version.
    uint64_t version = 1;
    mutable dbl::DevBuf digest;
    mutable uint64_t digest_version = 0;
};

namespace dbl {
// A CUB device call is two calls: a temporary-storage size query, which runs
// the whole host-side dispatch (occupancy queries; ~40 us of host time for a
// radix sort on this box), then the real one.  The size depends only on the
// call and its sizes, so it is cached per graph under (tag, a, b):
// call(tmp, bytes) must issue the CUB call.
template <class F>
dbl_status cub_cached(dbl_graph *g, int tag, uint64_t a, uint64_t b, F &&call) {
    const auto key = std::make_tuple(tag, a, b);
    size_t tmp = 0;
    auto it = g->cub_sizes.find(key);
    if (it == g->cub_sizes.end()) {
        cudaError_t e = call((void *)nullptr, tmp);
        if (e != cudaSuccess) return cuda_fail(e, "CUB temporary-size query");
        if (g->cub_sizes.size() > 4096) g->cub_sizes.clear();
        g->cub_sizes[key] = tmp;
    } else {
        tmp = it->second;
    }
    dbl_status s = g->cub_tmp.ensure(tmp);
    if (s) return s;
    cudaError_t e = call(g->cub_tmp.p, tmp);
    if (e != cudaSuccess) return cuda_fail(e, "CUB call");
    DBL_LAUNCHED();
    return DBL_OK;
}
enum { CUB_SORT = 1, CUB_UNIQUE = 2, CUB_FLAGGED = 3, CUB_SCAN = 4 };

// graph.cu
dbl_status graph_ensure_traversal(dbl_graph *g);
dbl_status graph_degrees_dev(const dbl_graph *g, uint32_t *indeg, uint32_t *outdeg);
Adj graph_fwd(const dbl_graph *g);
Adj graph_rev(const dbl_graph *g);
dbl_status build_csr_from_sorted(dbl_graph *g, const uint64_t *keys, uint64_t m, uint32_t n,
                                 uint32_t *ptr, uint32_t *col, const uint64_t *madd = nullptr,
                                 uint64_t madd_ub = 0);
dbl_status sort_keys_replay(dbl_graph *g, uint64_t *keys, uint64_t *alt, uint64_t m, int end_bit,
                            uint64_t **sorted);
dbl_status sort_keys(dbl_graph *g, uint64_t *keys, uint64_t *alt, uint64_t m, int end_bit,
                     uint64_t **sorted);
int key_end_bit(uint32_t n);
// dcount (optional): the number of new keys lives on the device and `count`
// is an upper bound; the caller settles g->m_delta after its final sync
dbl_status graph_insert_delta(dbl_graph *g, const uint64_t *new_keys_f, uint64_t count,
                              const uint64_t *dcount = nullptr);
dbl_status graph_filter_new(dbl_graph *g, const uint64_t *keys, uint64_t count, uint64_t *out,
                            uint64_t *nout, const uint64_t **dcount = nullptr,
                            const uint64_t *valid_dev = nullptr, const unsigned long long *abort_dev = nullptr);
dbl_status graph_compact(dbl_graph *g);
// Fold the single-edge pending log into the delta adjacency (every entry
// point that reads the adjacency or changes the graph calls this first).
constexpr uint32_t PEND_CAP = 1024;
dbl_status graph_flush_pending(dbl_graph *g);
// insert_one.cu: single-edge insert in one launch (done = false: the caller
// finishes with the batch fixpoint; the edge is already in the pending log)
dbl_status insert_edge_fast(dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v, dbl_update_stats *st,
                            bool *done, uint32_t *dirs_done, bool digest_current = false);
struct OneOut;
dbl_status insert_edge_outcome(dbl_graph *g, const OneOut &o, dbl_update_stats *st, bool *done,
                               uint32_t *dirs_done);
// select.cu
dbl_status select_landmarks_dev(dbl_graph *g, uint32_t k, int strategy, uint32_t *dev_out);
dbl_status select_leaves_dev(dbl_graph *g, uint64_t threshold, uint32_t k_prime, uint64_t seed,
                             const uint32_t *dev_ovr, uint8_t *dev_flags, uint32_t *dev_bucket);
dbl_status leaf_hash_dev(const uint64_t *ids, uint64_t count, uint32_t k_prime, uint64_t seed,
                         uint32_t *out, cudaStream_t s);
// Fused build prep: one pass over the vertices selects the leaves (if
// idx->sel_leaves), scores + histograms the landmark candidates (if
// idx->sel_landmarks), seeds every record word and writes the level-0
// frontier bitmaps bits0/bits1 for the record words [a0, e0) / [a1, e1);
// then the landmark top-k runs on the device and ORs the landmark bits into
// the records and the bitmaps.  No host synchronisation.
dbl_status prep_build_dev(dbl_graph *g, dbl_index *idx, uint32_t *bits0, uint32_t *bits1, uint32_t a0,
                          uint32_t e0, uint32_t a1, uint32_t e1, bool write_rec = true, uint32_t *haspred = nullptr, bool *haspred_written = nullptr);
// Enqueue the D2H copy of the prep state (read after the build's sync):
// err = bucket override outside [0, k'); fallback = the device top-k
// overflowed its candidate table (the caller re-selects and rebuilds).
dbl_status prep_fetch(dbl_graph *g, PrepState *host);
// fixpoint.cu
dbl_status index_seed_records(dbl_graph *g, dbl_index *idx, uint64_t wmask);
dbl_status run_build(dbl_graph *g, dbl_index *idx, const uint32_t *words, uint32_t nwords);
dbl_status run_insert(dbl_graph *g, dbl_index *idx, const uint64_t *new_keys, uint64_t count,
                      bool count_changes, uint32_t *changed_out, uint32_t *seed_changed,
                      uint32_t *levels, const unsigned long long *extra_dev = nullptr,
                      unsigned long long *extra_host = nullptr, const uint64_t *dcount = nullptr);
dbl_status work_model(const dbl_index *idx, dbl_graph *g, uint64_t *V, uint64_t *E,
                      uint32_t *levels);
// query.cu
void query_timings(dbl_graph *g);
// host_result: the closing CTA also writes the result words into the pinned
// g->q_host_res (synchronous calls read them there after the stream sync)
// host_inputs: u / v are pinned host memory read over PCIe (zero-copy)
dbl_status run_query(const dbl_index *idx, dbl_graph *g, const uint32_t *u, const uint32_t *v,
                     uint64_t count, uint32_t flags, uint8_t *codes, uint32_t *visited, bool host_result = false,
                     bool host_inputs = false);
dbl_status ensure_dense(const dbl_index *idx, dbl_graph *g);
dbl_status query_finish(dbl_graph *g, uint32_t *err_out, bool *dense_out);
dbl_status query_err_to(dbl_graph *g, uint32_t *dst4);
bool chunk_needs_dense(const uint32_t *w4);
dbl_status query_sync(dbl_graph *g);
// Stop every running per-call service (a no-op while none runs).
void serve_quiesce();
// While one exists (any thread), no per-call service runs or starts: every
// ABI entry except the single-call paths holds one for its duration, so no
// service runs beside a label or adjacency write, a cooperative launch or a
// handle release.
struct ServeBlock {
    ServeBlock();
    ~ServeBlock();
    ServeBlock(const ServeBlock &) = delete;
    ServeBlock &operator=(const ServeBlock &) = delete;
};
// Answer one host query through the service; *served = false: take the batch path.
dbl_status serve_query(const dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v, uint32_t flags, uint8_t *code,
                       uint32_t *visited, bool *served);
void serve_release(dbl_graph *g);
// Run one single-edge insert (K9) on the service.  *served = false: the
// caller launches K9 itself.  Otherwise the label version has moved, the
// outcome is in st / done / dirs_done as from insert_edge_fast, and *dig_ok
// tells whether the digest was current before the edge (for the fallback).
dbl_status serve_insert(dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v, dbl_update_stats *st, bool *done,
                        uint32_t *dirs_done, bool *dig_ok, bool *served);
// (Re)compute idx's digest on g's stream if it is stale (no host sync).
dbl_status digest_refresh(const dbl_index *idx, dbl_graph *g);
// After run_insert (count_changes): if the digest was current before the
// batch, recompute it for the vertices in the change bitmaps and mark it
// current again.
dbl_status digest_after_insert(dbl_index *idx, dbl_graph *g, bool was_current);
}  // namespace dbl
