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
// The counts are the reference's: visited = dequeues = 1 + changed
// non-seed vertices per direction, labels_changed = changed vertices
// (the seed when `add` was new to it).
//
// The pending log: single inserts append their edge here instead of
// rebuilding the delta CSR/CSC (O(n) per edge); later single inserts see
// the logged edges through a scan, and every other operation that reads the
// adjacency first folds the log into the delta (graph_flush_pending).
#include <cstring>

#include "internal.cuh"

namespace dbl {

constexpr int ONE_THREADS = 512;
constexpr int ONE_HCAP = 4096;        // discovered-vertex hash (power of two)
constexpr int ONE_FCAP = 2048;        // frontier list capacity per level
constexpr uint32_t ONE_EMAX = 1u << 16;   // adjacency entries scanned per direction before giving up
constexpr uint32_t ONE_EMPTY = 0xffffffffu;

struct OneOut {
    uint32_t certified;   // pre-check certified u -> v (early_terminated)
    uint32_t is_new;      // the edge was absent (appended to the pending log)
    uint32_t overflow;    // a cone outgrew the CTA tables: labels untouched
    uint32_t visited;
    uint32_t changed;
    uint32_t range;       // a discovered id was outside [0, n) (corrupt adjacency)
    uint32_t dirs_done;   // directions propagated and written (0, 1 or 2)
    uint32_t visited0, changed0;   // direction 0's counts (kept when direction 1 overflows)
};

struct OneShared {
    uint32_t key[ONE_HCAP];
    uint16_t lvl[ONE_HCAP];
    uint32_t front[2][ONE_FCAP];
    uint32_t nfront[2];
    uint32_t found;        // vertices discovered (non-seed)
    uint32_t edges;        // adjacency entries scanned
    uint32_t overflow;
    uint32_t exists;
    uint64_t add[2 * MAX_SHARD_WORDS];
};

__device__ __forceinline__ bool row_has(const uint32_t *ptr, const uint32_t *col, uint32_t u, uint32_t v) {
    if (!ptr) return false;
    uint32_t lo = ptr[u], hi = ptr[u + 1];
    while (lo < hi) {   // rows are sorted (built from sorted keys)
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t c = col[mid];
        if (c == v) return true;
        if (c < v) lo = mid + 1; else hi = mid;
    }
    return false;
}

// Insert x into the discovered set at level `l`; returns 1 if this call
// inserted it, 0 if present, -1 if the table is full.
__device__ __forceinline__ int one_insert(OneShared &S, uint32_t x, uint16_t l) {
    uint32_t h = (x * 0x9E3779B1u) >> 20;   // 12 bits
#pragma unroll 1
    for (int p = 0; p < 64; ++p) {
        const uint32_t k = S.key[h];
        if (k == x) return 0;
        if (k == ONE_EMPTY) {
            const uint32_t old = atomicCAS(&S.key[h], ONE_EMPTY, x);
            if (old == ONE_EMPTY) { S.lvl[h] = l; return 1; }
            if (old == x) return 0;
        }
        h = (h + 1) & (ONE_HCAP - 1);
    }
    return -1;
}

__device__ __forceinline__ int one_find(const OneShared &S, uint32_t x) {
    uint32_t h = (x * 0x9E3779B1u) >> 20;
#pragma unroll 1
    for (int p = 0; p < 64; ++p) {
        const uint32_t k = *(volatile const uint32_t *)&S.key[h];
        if (k == x) return (int)h;
        if (k == ONE_EMPTY) return -1;
        h = (h + 1) & (ONE_HCAP - 1);
    }
    return -1;
}

// Does x's half (H words at rec + x * rs + off) lack some bit of S.add?
__device__ __forceinline__ bool lacks(const uint64_t *rec, uint32_t rs, uint32_t off, uint32_t H, uint32_t x,
                                      const uint64_t *add) {
    const uint64_t *p = rec + (uint64_t)x * rs + off;
    uint64_t m = 0;
    for (uint32_t j = 0; j < H; ++j) m |= add[j] & ~__ldg(p + j);
    return m != 0;
}

__device__ void one_consider(OneShared &S, const uint64_t *rec, uint32_t rs, uint32_t off, uint32_t H, uint32_t n,
                             uint32_t x, uint16_t nl, uint32_t *range) {
    if (x >= n) { *range = 1; S.overflow = 1; return; }
    if (one_find(S, x) >= 0) return;
    if (!lacks(rec, rs, off, H, x, S.add)) return;
    const int r = one_insert(S, x, nl);
    if (r < 0) { S.overflow = 1; return; }
    if (r == 1) {
        const uint32_t p = atomicAdd(&S.nfront[nl & 1], 1u);
        if (p >= ONE_FCAP) { S.overflow = 1; return; }
        S.front[nl & 1][p] = x;
        atomicAdd(&S.found, 1u);
    }
}

// One direction: seed s, add = the other endpoint's half, labels at word
// offset `off` of each record, neighbours along `a` plus the pending edges
// (fwd: entries (s', t) with s' in the frontier give t; bwd: (t, s') give t).
// Returns the number of discovered non-seed vertices (S.overflow on failure).
__device__ uint32_t one_direction(OneShared &S, const uint64_t *rec, uint32_t rs, uint32_t off, uint32_t H,
                                  uint32_t n, const Adj &a, const uint64_t *pend, uint32_t npend, bool fwd,
                                  uint32_t seed, uint32_t *range) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = ONE_THREADS / 32;
    for (int i = tid; i < ONE_HCAP; i += ONE_THREADS) S.key[i] = ONE_EMPTY;
    if (tid == 0) {
        S.nfront[0] = 1;
        S.nfront[1] = 0;
        S.front[0][0] = seed;
        S.found = 0;
        S.edges = 0;
    }
    __syncthreads();
    if (tid == 0) one_insert(S, seed, 0);   // the seed is expanded once and never re-enqueued
    __syncthreads();
    for (uint16_t l = 0;; ++l) {
        const int cb = l & 1, nb = cb ^ 1;
        const uint32_t nf = min(S.nfront[cb], (uint32_t)ONE_FCAP);
        if (nf == 0 || S.overflow) break;
        // adjacency rows of the frontier: a warp per vertex, lanes over the row
        for (uint32_t i = warp; i < nf; i += nwarps) {
            const uint32_t p = S.front[cb][i];
#pragma unroll 1
            for (int seg = 0; seg < 2; ++seg) {
                const uint32_t *ptr = seg ? a.dptr : a.ptr;
                if (!ptr) break;
                const uint32_t *col = seg ? a.dcol : a.col;
                const uint32_t s0 = __ldg(ptr + p), s1 = __ldg(ptr + p + 1);
                int stop = 0;
                if (lane == 0) {
                    if (atomicAdd(&S.edges, s1 - s0) + (s1 - s0) > ONE_EMAX) S.overflow = 1;
                    stop = *(volatile uint32_t *)&S.overflow != 0;
                }
                if (__shfl_sync(FULL, stop, 0)) break;   // warp-uniform
                for (uint32_t j = s0 + lane; j < s1; j += 32)
                    one_consider(S, rec, rs, off, H, n, __ldg(col + j), (uint16_t)(l + 1), range);
            }
        }
        // pending edges leaving (fwd) / entering (bwd) a vertex of this level
        for (uint32_t e = tid; e < npend; e += ONE_THREADS) {
            const uint64_t k = pend[e];
            const uint32_t from = fwd ? (uint32_t)(k >> 32) : (uint32_t)k;
            const uint32_t to = fwd ? (uint32_t)k : (uint32_t)(k >> 32);
            const int sl = one_find(S, from);
            if (sl >= 0 && S.lvl[sl] == l) one_consider(S, rec, rs, off, H, n, to, (uint16_t)(l + 1), range);
        }
        __syncthreads();
        if (tid == 0) S.nfront[cb] = 0;
        __syncthreads();
        (void)nb;
    }
    __syncthreads();
    return S.found;
}

// OR S.add into the discovered vertices' halves (and the seed's).
__device__ void one_apply(OneShared &S, uint64_t *rec, uint32_t rs, uint32_t off, uint32_t H) {
    for (int i = threadIdx.x; i < ONE_HCAP; i += ONE_THREADS) {
        const uint32_t x = S.key[i];
        if (x == ONE_EMPTY) continue;
        uint64_t *p = rec + (uint64_t)x * rs + off;
        for (uint32_t j = 0; j < H; ++j) p[j] |= S.add[j];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(ONE_THREADS, 1)
insert_one_kernel(uint64_t *rec, uint32_t rs, uint32_t H, uint32_t wdl, uint32_t n, uint32_t u, uint32_t v,
                  Adj fwd, Adj rev, uint64_t *pend, uint32_t npend, uint32_t pcap, OneOut *out) {
    extern __shared__ __align__(16) unsigned char smem[];
    OneShared &S = *reinterpret_cast<OneShared *>(smem);
    const int tid = threadIdx.x;
    const uint64_t key = ((uint64_t)u << 32) | v;
    __shared__ uint32_t cert, range;
    if (tid == 0) {
        // pre-check on pre-insertion labels (updates.py:123)
        uint64_t c = 0;
        for (uint32_t j = 0; j < wdl; ++j) c |= rec[(uint64_t)u * rs + H + j] & rec[(uint64_t)v * rs + j];
        cert = c != 0;
        range = 0;
        S.overflow = 0;
        S.exists = row_has(fwd.ptr, fwd.col, u, v) || row_has(fwd.dptr, fwd.dcol, u, v);
    }
    __syncthreads();
    for (uint32_t e = tid; e < npend; e += ONE_THREADS)
        if (pend[e] == key) S.exists = 1;
    __syncthreads();
    const bool is_new = !S.exists;
    if (tid == 0 && is_new && npend < pcap) pend[npend] = key;   // add_edge (updates.py:124)
    OneOut o{};
    o.certified = cert;
    o.is_new = is_new;
    if (!cert) {
        // forward from v with L_in(u) (updates.py:128-130), then backward from u
        // with L_out(v) (:131-133); the halves are {dl | bl} at offsets 0 and H
        uint32_t changed = 0, visited = 0;
        bool ok = true;
        for (int d = 0; d < 2 && ok; ++d) {
            const uint32_t seed = d == 0 ? v : u, other = d == 0 ? u : v, off = d == 0 ? 0 : H;
            for (uint32_t j = tid; j < H; j += ONE_THREADS) S.add[j] = rec[(uint64_t)other * rs + off + j];
            __syncthreads();
            const bool seed_changes = lacks(rec, rs, off, H, seed, S.add);
            const uint32_t found = one_direction(S, rec, rs, off, H, n, d == 0 ? fwd : rev, pend,
                                                 npend + ((is_new && npend < pcap) ? 1 : 0), d == 0, seed, &range);
            if (S.overflow) { ok = false; break; }
            // the directions touch disjoint words (in- vs out-half), so each is
            // written as soon as its cone is known; when direction 1 then
            // overflows, the host finishes only that one (dirs_done = 1)
            one_apply(S, rec, rs, off, H);
            visited += 1 + found;
            changed += found + (seed_changes ? 1 : 0);
            o.dirs_done = d + 1;
            if (d == 0) { o.visited0 = visited; o.changed0 = changed; }
        }
        o.overflow = !ok;
        o.visited = visited;
        o.changed = changed;
    }
    if (tid == 0) {
        o.range = range;
        *out = o;
        __threadfence_system();
    }
}

}  // namespace dbl

using namespace dbl;

namespace dbl {

// Single-edge insert, fast path.  Returns DBL_OK with *done = false when the
// caller must finish with the batch fixpoint: a cone outgrew the tables; the
// edge is in the pending log, direction 0 is finished (labels written, counts
// in *st) iff *dirs_done == 1, and direction 1 is untouched.
dbl_status insert_edge_fast(dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v, dbl_update_stats *st,
                            bool *done, uint32_t *dirs_done) {
    *done = false;
    *dirs_done = 0;
    dbl_status s;
    if (g->n_pend >= PEND_CAP && (s = graph_flush_pending(g))) return s;
    if ((s = g->pend.ensure(PEND_CAP * 8 + 64)) || (s = g->one_out.ensure(sizeof(OneOut) + 64))) return s;
    if (idx->wdl + idx->wbl > (uint32_t)MAX_SHARD_WORDS) { set_error("label width too large"); return DBL_E_CONFIG; }
    int bps = 1;
    if ((s = kernel_occupancy((const void *)insert_one_kernel, ONE_THREADS, sizeof(OneShared), &bps))) return s;
    OneOut *out = reinterpret_cast<OneOut *>(g->one_out.p);
    insert_one_kernel<<<1, ONE_THREADS, sizeof(OneShared), g->stream>>>(
        idx->rec.as<uint64_t>(), idx->rs, idx->wdl + idx->wbl, idx->wdl, g->n, u, v, graph_fwd(g), graph_rev(g),
        g->pend.as<uint64_t>(), g->n_pend, PEND_CAP, out);
    DBL_CHECK_LAUNCH("insert_one_kernel");
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    OneOut o;
    std::memcpy(&o, out, sizeof(o));
    if (o.range) { set_error("adjacency holds a vertex outside [0, n)"); return DBL_E_CUDA; }
    if (o.is_new) ++g->n_pend;
    st->inserted = o.is_new;
    if (o.certified) {
        st->early_terminated = 1;
        *done = true;
        return DBL_OK;
    }
    if (o.overflow) {   // direction 0 may be done: its counts stand
        st->visited = o.dirs_done ? o.visited0 : 0;
        st->labels_changed = o.dirs_done ? o.changed0 : 0;
        *dirs_done = o.dirs_done;
        return DBL_OK;
    }
    st->visited = o.visited;
    st->labels_changed = o.changed;
    *done = true;
    return DBL_OK;
}

}  // namespace dbl
