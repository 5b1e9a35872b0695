// insert_one.cuh -- device code of the single-edge insert (K9), shared by
// insert_one.cu (one launch per call) and the per-call service (query.cu).
// See insert_one.cu for the algorithm and its reference lines.
#pragma once

#include "internal.cuh"

namespace dbl {

constexpr int ONE_THREADS = 512;
constexpr int ONE_HALF = ONE_THREADS / 2;   // threads per direction (the two run concurrently)
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
    uint32_t done[2];     // direction d propagated and written
    uint32_t dvisited[2], dchanged[2];   // per-direction counts (kept when the other overflows)
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

// Warp-cooperative search of a sorted row: 32 probes per step narrow the
// interval 32-fold (a hub's row of 10^5 ids takes 3 steps, not 17).
static __device__ __forceinline__ bool row_has_warp(const uint32_t *ptr, const uint32_t *col, uint32_t u, uint32_t v) {
    if (!ptr) return false;
    const int lane = threadIdx.x & 31;
    uint32_t lo = ptr[u], hi = ptr[u + 1];   // candidates [lo, hi)
    while (hi - lo > 32) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t p = lo + lane * step;
        const bool le = p < hi && col[p] <= v;
        const unsigned b = __ballot_sync(FULL, le);
        const uint32_t k = b ? 31 - __clz(b) : 0;   // last probe <= v
        if (!b) return false;
        lo = lo + k * step;
        hi = min(hi, lo + step);
    }
    const bool hit = lo + lane < hi && col[lo + lane] == v;
    return __any_sync(FULL, hit);
}

// Insert x into the discovered set at level `l`; returns 1 if this call
// inserted it, 0 if present, -1 if the table is full.
static __device__ __forceinline__ int one_insert(OneShared &S, uint32_t x, uint16_t l) {
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

static __device__ __forceinline__ int one_find(const OneShared &S, uint32_t x) {
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
static __device__ __forceinline__ bool lacks(const uint64_t *rec, uint32_t rs, uint32_t off, uint32_t H, uint32_t x,
                                      const uint64_t *add) {
    const uint64_t *p = rec + (uint64_t)x * rs + off;
    uint64_t m = 0;
    for (uint32_t j = 0; j < H; ++j) m |= add[j] & ~__ldcg(p + j);   // not .nc: the service writes records
    return m != 0;
}

static __device__ void one_consider(OneShared &S, const uint64_t *rec, uint32_t rs, uint32_t off, uint32_t H, uint32_t n,
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

// barrier of one direction's half of the CTA (named barriers 1 and 2)
static __device__ __forceinline__ void half_sync(int h) {
    asm volatile("bar.sync %0, %1;" ::"r"(h + 1), "r"(ONE_HALF) : "memory");
}

// One direction: seed s, add = the other endpoint's half, labels at word
// offset `off` of each record, neighbours along `a` plus the pending edges
// (fwd: entries (s', t) with s' in the frontier give t; bwd: (t, s') give t).
// Returns the number of discovered non-seed vertices (S.overflow on failure).
static __device__ uint32_t one_direction(OneShared &S, const uint64_t *rec, uint32_t rs, uint32_t off, uint32_t H,
                                  uint32_t n, const Adj &a, const uint64_t *pend, uint32_t npend, bool fwd,
                                  uint32_t seed, uint32_t *range, int h) {
    const int tid = threadIdx.x - h * ONE_HALF, lane = tid & 31, warp = tid >> 5, nwarps = ONE_HALF / 32;
    for (int i = tid; i < ONE_HCAP; i += ONE_HALF) S.key[i] = ONE_EMPTY;
    if (tid == 0) {
        S.nfront[0] = 1;
        S.nfront[1] = 0;
        S.front[0][0] = seed;
        S.found = 0;
        S.edges = 0;
    }
    half_sync(h);
    if (tid == 0) one_insert(S, seed, 0);   // the seed is expanded once and never re-enqueued
    half_sync(h);
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
        for (uint32_t e = tid; e < npend; e += ONE_HALF) {
            const uint64_t k = pend[e];
            const uint32_t from = fwd ? (uint32_t)(k >> 32) : (uint32_t)k;
            const uint32_t to = fwd ? (uint32_t)k : (uint32_t)(k >> 32);
            const int sl = one_find(S, from);
            if (sl >= 0 && S.lvl[sl] == l) one_consider(S, rec, rs, off, H, n, to, (uint16_t)(l + 1), range);
        }
        half_sync(h);
        if (tid == 0) S.nfront[cb] = 0;
        half_sync(h);
        (void)nb;
    }
    half_sync(h);
    return S.found;
}

static __device__ __forceinline__ uint32_t fold14_one(uint64_t x) {
    return (uint32_t)((x | (x >> 14) | (x >> 28) | (x >> 42) | (x >> 56)) & 0x3fffu);
}

// OR S.add into the discovered vertices' halves (and the seed's).  With a
// query digest (query.cu: each digest bit is the OR of a fixed set of label
// bits), the digest bits of S.add are ORed into the same vertices' digests,
// which keeps a current digest exact.
static __device__ void one_apply(OneShared &S, uint64_t *rec, uint32_t rs, uint32_t off, uint32_t H, uint32_t wdl,
                          uint32_t *dig, int h) {
    uint32_t dm = 0;
    if (dig) {
        if (wdl) {
            uint64_t rest = S.add[0] & ~1ull;
            for (uint32_t j = 1; j < wdl; ++j) rest |= S.add[j];
            dm = (uint32_t)(S.add[0] & 1u) | (rest ? 2u : 0u);
        }
        uint32_t f = 0;
        for (uint32_t j = wdl; j < H; ++j) f |= fold14_one(S.add[j]);
        // in-half (h = 0): dl_in -> bits 2, 3, bl_in -> 4..17; out-half: dl_out -> 0, 1, bl_out -> 18..31
        dm = h == 0 ? (dm << 2) | (f << 4) : dm | (f << 18);
    }
    for (int i = threadIdx.x - h * ONE_HALF; i < ONE_HCAP; i += ONE_HALF) {
        const uint32_t x = S.key[i];
        if (x == ONE_EMPTY) continue;
        uint64_t *p = rec + (uint64_t)x * rs + off;
        for (uint32_t j = 0; j < H; ++j) p[j] |= S.add[j];
        if (dm) atomicOr(dig + x, dm);
    }
    half_sync(h);
}

// The whole single-edge insert, run by a CTA of ONE_THREADS threads with two
// OneShared tables (one per direction) in shared memory: by insert_one_kernel
// (one launch per call) and by the per-call service kernel (query.cu).
static __device__ void insert_one_body(uint64_t *rec, uint32_t rs, uint32_t H, uint32_t wdl, uint32_t n, uint32_t u,
                                       uint32_t v, const Adj &fwd, const Adj &rev, uint64_t *pend, uint32_t npend,
                                       uint32_t pcap, OneOut *out, uint32_t *dig, OneShared *S2) {
    const int tid = threadIdx.x;
    const uint64_t key = ((uint64_t)u << 32) | v;
    __shared__ uint32_t cert, range, exists;
    __shared__ uint32_t rok[2], rvis[2], rchg[2];
    if (tid == 0) { range = 0; exists = 0; }
    __syncthreads();
    // in parallel: warp 0 the base row, warp 1 the delta row, warp 2 the
    // pre-check on pre-insertion labels (updates.py:123), the rest the log
    const int w = tid >> 5;
    if (w == 0) {
        if (row_has_warp(fwd.ptr, fwd.col, u, v) && (tid & 31) == 0) exists = 1;
    } else if (w == 1) {
        if (row_has_warp(fwd.dptr, fwd.dcol, u, v) && (tid & 31) == 0) exists = 1;
    } else if (w == 2) {
        if ((tid & 31) == 0) {
            uint64_t c = 0;
            for (uint32_t j = 0; j < wdl; ++j) c |= rec[(uint64_t)u * rs + H + j] & rec[(uint64_t)v * rs + j];
            cert = c != 0;
        }
    } else {
        for (uint32_t e = tid - 96; e < npend; e += ONE_THREADS - 96)
            if (pend[e] == key) exists = 1;
    }
    __syncthreads();
    const bool is_new = !exists;
    if (tid == 0 && is_new && npend < pcap) pend[npend] = key;   // add_edge (updates.py:124)
    if (!cert) {
        // both propagations at once, one per half of the CTA: forward from v
        // with L_in(u) (updates.py:128-130), backward from u with L_out(v)
        // (:131-133).  They read and write disjoint words (the in-half at
        // word 0, the out-half at word H of every record), so neither sees
        // the other's writes.
        const int h = tid / ONE_HALF, ltid = tid - h * ONE_HALF;
        OneShared &S = S2[h];
        const uint32_t seed = h == 0 ? v : u, other = h == 0 ? u : v, off = h == 0 ? 0 : H;
        for (uint32_t j = ltid; j < H; j += ONE_HALF) S.add[j] = rec[(uint64_t)other * rs + off + j];
        if (ltid == 0) S.overflow = 0;
        half_sync(h);
        const bool seed_changes = lacks(rec, rs, off, H, seed, S.add);
        const uint32_t found = one_direction(S, rec, rs, off, H, n, h == 0 ? fwd : rev, pend,
                                             npend + ((is_new && npend < pcap) ? 1 : 0), h == 0, seed, &range, h);
        const bool ok = !S.overflow;
        if (ok) one_apply(S, rec, rs, off, H, wdl, dig, h);
        if (ltid == 0) {
            rok[h] = ok;
            rvis[h] = 1 + found;
            rchg[h] = found + (seed_changes ? 1 : 0);
        }
    }
    __syncthreads();
    if (tid == 0) {
        OneOut o{};
        o.certified = cert;
        o.is_new = is_new;
        o.range = range;
        if (!cert) {
            o.overflow = !(rok[0] && rok[1]);
            for (int d = 0; d < 2; ++d) {
                o.done[d] = rok[d];
                o.dvisited[d] = rok[d] ? rvis[d] : 0;
                o.dchanged[d] = rok[d] ? rchg[d] : 0;
            }
            o.visited = o.dvisited[0] + o.dvisited[1];
            o.changed = o.dchanged[0] + o.dchanged[1];
        }
        *out = o;
    }
}

}  // namespace dbl
