// insert_one.cu -- single-edge insert_edge in one launch and one host sync.
//
// Reference: insert_edge (updates.py:112-137) and _propagate_union
// (updates.py:89-109).  One CTA does the whole call:
//   1. the pre-check dl_out[u] & dl_in[v] on pre-insertion labels (:123);
//   2. add_edge (:124): the edge is looked up in the base and delta
//      adjacency (binary search of the sorted rows) and in the graph's
//      pending-edge log, and appended to that log if new;
//   3. unless certified, both propagations (:129-134) as a discovery BFS
//      followed by one write pass.  With add = the seed-side half of the
//      other endpoint's record, the vertices _propagate_union changes are
//      exactly those reachable from the seed through vertices that lack
//      `add` (a vertex holding `add` blocks the cone, a changed vertex is
//      enqueued once), independent of the visiting order -- so discovery
//      reads labels only, and the labels are written only once the cone is
//      known to fit the CTA's tables.  A cone that outgrows them leaves that
//      direction's labels untouched and the host runs the batch fixpoint
//      (run_insert), counting only the directions the kernel did not finish.
//      The two directions run concurrently, one per half of the CTA.
// The counts are the reference's: visited = dequeues = 1 + changed
// non-seed vertices per direction, labels_changed = changed vertices
// (the seed when `add` was new to it).
//
// The pending log: single inserts append their edge here instead of
// rebuilding the delta CSR/CSC (O(n) per edge); later single inserts see
// the logged edges through a scan, and every other operation that reads the
// adjacency first folds the log into the delta (graph_flush_pending).
#include <cstring>

#include "insert_one.cuh"

namespace dbl {

__global__ void __launch_bounds__(ONE_THREADS, 1)
insert_one_kernel(uint64_t *rec, uint32_t rs, uint32_t H, uint32_t wdl, uint32_t n, uint32_t u, uint32_t v,
                  Adj fwd, Adj rev, uint64_t *pend, uint32_t npend, uint32_t pcap, OneOut *out, uint32_t *dig) {
    extern __shared__ __align__(16) unsigned char smem[];
    insert_one_body(rec, rs, H, wdl, n, u, v, fwd, rev, pend, npend, pcap, out, dig, reinterpret_cast<OneShared *>(smem));
}

}  // namespace dbl

using namespace dbl;

namespace dbl {

// Single-edge insert, fast path.  Returns DBL_OK with *done = false when the
// caller must finish with the batch fixpoint: a cone outgrew the tables; the
// edge is in the pending log, direction d is finished (labels written, its
// counts in *st) iff bit d of *dirs_done is set, the other is untouched.
dbl_status insert_edge_fast(dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v, dbl_update_stats *st,
                            bool *done, uint32_t *dirs_done, bool digest_current) {
    *done = false;
    *dirs_done = 0;
    dbl_status s;
    if (g->n_pend >= PEND_CAP && (s = graph_flush_pending(g))) return s;
    if ((s = g->pend.ensure(PEND_CAP * 8 + 64)) || (s = g->one_out.ensure(sizeof(OneOut) + 64))) return s;
    if (idx->wdl + idx->wbl > (uint32_t)MAX_SHARD_WORDS) { set_error("label width too large"); return DBL_E_CONFIG; }
    int bps = 1;
    if ((s = kernel_occupancy((const void *)insert_one_kernel, ONE_THREADS, 2 * sizeof(OneShared), &bps))) return s;
    OneOut *out = reinterpret_cast<OneOut *>(g->one_out.p);
    insert_one_kernel<<<1, ONE_THREADS, 2 * sizeof(OneShared), g->stream>>>(
        idx->rec.as<uint64_t>(), idx->rs, idx->wdl + idx->wbl, idx->wdl, g->n, u, v, graph_fwd(g), graph_rev(g),
        g->pend.as<uint64_t>(), g->n_pend, PEND_CAP, out, digest_current ? idx->digest.as<uint32_t>() : nullptr);
    DBL_CHECK_LAUNCH("insert_one_kernel");
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    OneOut o;
    std::memcpy(&o, out, sizeof(o));
    return insert_edge_outcome(g, o, st, done, dirs_done);
}

// K9's result -> UpdateStats; *done = false: a cone outgrew the tables and
// the caller finishes with the batch fixpoint (direction d is finished iff
// bit d of *dirs_done is set, its counts already in *st).
dbl_status insert_edge_outcome(dbl_graph *g, const OneOut &o, dbl_update_stats *st, bool *done,
                               uint32_t *dirs_done) {
    *done = false;
    *dirs_done = 0;
    if (o.range) { set_error("adjacency holds a vertex outside [0, n)"); return DBL_E_CUDA; }
    if (o.is_new) ++g->n_pend;
    st->inserted = o.is_new;
    if (o.certified) {
        st->early_terminated = 1;
        *done = true;
        return DBL_OK;
    }
    if (o.overflow) {   // a finished direction's counts stand
        st->visited = o.dvisited[0] + o.dvisited[1];
        st->labels_changed = o.dchanged[0] + o.dchanged[1];
        *dirs_done = (o.done[0] ? 1u : 0u) | (o.done[1] ? 2u : 0u);
        return DBL_OK;
    }
    st->visited = o.visited;
    st->labels_changed = o.changed;
    *done = true;
    return DBL_OK;
}

}  // namespace dbl
