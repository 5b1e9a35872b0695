// fixpoint.cu -- K3/K4 label construction and K8 insertion propagation.
//
// Reference: build_index (labels.py:263-306) floods one bit at a time with a
// BFS (_flood, labels.py:247-260); insert_edge (updates.py:112-137) ORs the
// new edge's labels through the affected cone (_propagate_union,
// updates.py:89-109).  Both compute the least fixpoint of
//     L[x] = seed[x] | OR_{p -> x} L[p]
// per label bit, which is unique, so any traversal order yields the
// reference's labels bit-for-bit.
//
// B200 design: all bits of a record half propagate together.  The in-half
// {dl_in, bl_in} (forward along CSR) and the out-half {dl_out, bl_out}
// (backward along CSC) run in ONE persistent cooperative kernel, one grid
// barrier per BFS level, no host round trip between levels.  Each level is
// split into equal edge ranges, one per warp (work items carry their offset
// in the level's edge space), so a hub's adjacency spreads over many warps
// and every warp relaxes 32 consecutive edges per step regardless of the
// degree mix.  A relaxed edge reads the destination's words through L2 and
// issues atomicOr only for the missing bits; a vertex whose label grew is
// stamped (one enqueue per level) and its edge ranges appended with a
// warp-aggregated atomicAdd.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace cg = cooperative_groups;

// Variant switches (build.build_variant -D flags; defaults = measured best)
#ifndef DBL_FIX_BPS_BUILD
#define DBL_FIX_BPS_BUILD 0      // fixpoint CTAs/SM for builds (0 = occupancy maximum)
#endif
#ifndef DBL_FIX_BPS_INSERT
#define DBL_FIX_BPS_INSERT 2     // fixpoint CTAs/SM for insert batches
#endif
#ifndef DBL_PULL_DIV
#define DBL_PULL_DIV 0u          // pull levels when frontier edges > m / d (0: push only)
#endif
#ifndef DBL_NO_PIVOT
#define DBL_NO_PIVOT 0           // 1: no pivot head start (plain fixpoint from the seeds)
#endif
#ifndef DBL_TD_DIV
#define DBL_TD_DIV 64u           // pivot reach: top-down once a step marks < n / d
#endif
#ifndef DBL_COMPACT_SLICES
#define DBL_COMPACT_SLICES 0     // 1: each warp compacts one contiguous slice of the bitmap
#endif
#ifndef DBL_PREP_RECORDS
#define DBL_PREP_RECORDS 0       // 1: prep writes the seeded records even when the pivot could
#endif

namespace dbl {

__device__ __forceinline__ uint64_t ld_cg64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void ld_cg128(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
__device__ __forceinline__ uint32_t ld_cg32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ void ld_cg256(const uint64_t *p, uint64_t &a, uint64_t &b, uint64_t &c, uint64_t &d) {
    asm volatile("ld.global.cg.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

template <int NW, int AL>
__device__ __forceinline__ void load_chunked(const uint64_t *p, uint64_t (&w)[NW]) {
    const uint64_t *b = p - AL;
    uint64_t c0, c1, c2, c3;
    ld_cg256(b, c0, c1, c2, c3);
    const uint64_t lo[4] = {c0, c1, c2, c3};
#pragma unroll
    for (int k = 0; k < NW && k + AL < 4; ++k) w[k] = lo[k + AL];
    if constexpr (AL + NW > 4) {
        ld_cg256(b + 4, c0, c1, c2, c3);
        const uint64_t hi[4] = {c0, c1, c2, c3};
#pragma unroll
        for (int k = 4 - AL; k < NW; ++k) w[k] = hi[k + AL - 4];
    }
}

// NW label words at p.  `al` (warp-uniform, from DirParams) is p's offset in
// words inside a 32-byte chunk when the record stride keeps chunks aligned,
// else -1.  5-word groups (the k = 256, k' = 64 halves) then load the covering
// 32-byte chunks -- two requests instead of one per word: random label reads
// are bound by L1->L2 requests, not bytes (tools/ubench_gather.cu).
template <int NW, bool VEC>
__device__ __forceinline__ void load_words(const uint64_t *p, uint64_t (&w)[NW], int al) {
    if constexpr (NW == 5) {   // (3- and 4-word groups spill at 64 registers with the 4-way switch)
        if (al >= 0) {
            switch (al) {   // warp-uniform; compile-time register indices in each case
            case 0: load_chunked<NW, 0>(p, w); return;
            case 1: load_chunked<NW, 1>(p, w); return;
            case 2: load_chunked<NW, 2>(p, w); return;
            default: load_chunked<NW, 3>(p, w); return;
            }
        }
    }
    if constexpr (VEC && (NW % 2 == 0)) {
#pragma unroll
        for (int k = 0; k < NW; k += 2) ld_cg128(p + k, w[k], w[k + 1]);
    } else {
#pragma unroll
        for (int k = 0; k < NW; ++k) w[k] = ld_cg64(p + k);
    }
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ uint32_t warp_excl_scan_u32(uint32_t x, uint32_t &total) {
    const uint32_t incl = warp_incl_scan(x);
    total = __shfl_sync(FULL, incl, 31);
    return incl - x;
}

// position of the r-th (0-based) set bit of mask
__device__ __forceinline__ int select_bit(uint32_t mask, uint32_t r) {
    int p = 0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        uint32_t low = mask & ((1u << s) - 1u);
        uint32_t c = __popc(low);
        if (r >= c) { r -= c; mask >>= s; p += s; } else { mask = low; }
    }
    return p;
}

// Append the adjacency segments of every lane's vertex y (if p) to queue QN:
// one warp-aggregated 64-bit atomicAdd reserves both the item slots and the
// edge-space offsets, so eoff stays monotone in the item index.
__device__ __forceinline__ void warp_enqueue(const DirParams &D, const Queue &QN, bool p, uint32_t y,
                                             unsigned long long *cnt_ptr, Ctrl *ctrl) {
    const int lane = threadIdx.x & 31;
    uint32_t b0 = 0, b1 = 0, d0 = 0, d1 = 0;
    if (p) {
        b0 = __ldg(D.adj.ptr + y);
        b1 = __ldg(D.adj.ptr + y + 1);
        if (D.adj.dptr) {
            d0 = __ldg(D.adj.dptr + y);
            d1 = __ldg(D.adj.dptr + y + 1);
        }
    }
    const uint32_t ni = (b1 > b0) + (d1 > d0);
    const uint32_t ne = (b1 - b0) + (d1 - d0);
    const uint32_t ii = warp_incl_scan(ni), ei = warp_incl_scan(ne);
    const uint32_t ti = __shfl_sync(FULL, ii, 31), te = __shfl_sync(FULL, ei, 31);
    if (ti == 0) return;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(cnt_ptr, ((unsigned long long)ti << 32) | te);
    base = __shfl_sync(FULL, base, 31);
    const uint32_t ibase = (uint32_t)(base >> 32), ebase = (uint32_t)base;
    if ((uint64_t)ibase + ti > D.cap) {
        if (lane == 0) atomicOr(&ctrl->overflow, 1u);
        return;
    }
    uint32_t pos = ibase + ii - ni, eo = ebase + ei - ne;
    if (b1 > b0) {
        QN.x[pos] = y; QN.start[pos] = b0; QN.len[pos] = b1 - b0; QN.eoff[pos] = eo;
        ++pos;
        eo += b1 - b0;
    }
    if (d1 > d0) {
        QN.x[pos] = y; QN.start[pos] = d0; QN.len[pos] = (d1 - d0) | DELTA_BIT; QN.eoff[pos] = eo;
    }
}

__device__ __forceinline__ void red_or(uint64_t *p, uint64_t v) {
    asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_or32(uint32_t *p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// OR the source words into y's words, marking y in the next-level bitmap when
// its (L2-coherent) read lacked bits; true iff anything was missing.
template <int NW, bool VEC>
__device__ __forceinline__ bool relax_mark(const DirParams &D, uint32_t y, const uint64_t (&s)[NW]) {
    uint64_t *p = D.lab + (size_t)y * D.stride;
    uint64_t c[NW];
    load_words<NW, VEC>(p, c, D.al);
    bool ch = false;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const uint64_t need = s[k] & ~c[k];
        if (need) { red_or(p + k, need); ch = true; }
    }
    if (ch) red_or32(D.bits + (y >> 5), 1u << (y & 31));
    return ch;
}

// Last item whose edge offset is <= e, searching [lo, nitems) 32-ary.
__device__ __forceinline__ uint32_t find_item(const uint32_t *eoff, uint32_t lo, uint32_t nitems, uint32_t e) {
    const int lane = threadIdx.x & 31;
    uint32_t hi = nitems;  // invariant: eoff[lo] <= e < eoff[hi] (eoff[nitems] = inf)
    while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t idx = lo + lane * step;
        const bool le = idx < hi && ld_cg32(eoff + idx) <= e;
        const unsigned bal = __ballot_sync(FULL, le);
        const uint32_t k = 31 - __clz(bal);
        lo += k * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

// Phase A: one warp relaxes the edges [e0, e1) of a level's edge space, U
// rounds of 32 consecutive edges at a time.  Each lane finds its item in a
// 32-item window by a 5-step shuffle search (the window slides forward as
// edges are consumed); the U column loads, the U destination reads and the
// fire-and-forget ORs (labels + next-frontier bitmap) are issued back to back
// so their latencies overlap.  Nothing waits on an atomic result.
template <int NW, bool VEC>
__device__ __forceinline__ void expand_range(const DirParams &D, uint32_t nitems, uint32_t e0, uint32_t e1) {
#ifndef DBL_FU
#define DBL_FU 2
#endif
    constexpr int U = NW <= 2 ? DBL_FU : (NW <= 4 ? 2 : 1);
    const Queue &Q = D.q;
    const int lane = threadIdx.x & 31;
    uint32_t i0 = find_item(Q.eoff, 0, nitems, e0);
    uint32_t wE = 0xffffffffu, wS = 0, wEnd = 0, winEnd = 0;
    int wD = 0;
    uint64_t w[NW];
    auto load_window = [&](uint32_t first) {
        const uint32_t i = first + lane;
        if (i < nitems) {
            wE = ld_cg32(Q.eoff + i);
            wS = ld_cg32(Q.start + i);
            const uint32_t lf = ld_cg32(Q.len + i);
            const uint32_t x = ld_cg32(Q.x + i);
            wD = (lf & DELTA_BIT) ? 1 : 0;
            wEnd = wE + (lf & ~DELTA_BIT);
            load_words<NW, VEC>(D.lab + (size_t)x * D.stride, w, D.al);
        } else {
            wE = 0xffffffffu;
            wEnd = 0;
#pragma unroll
            for (int k = 0; k < NW; ++k) w[k] = 0;
        }
        const unsigned valid = __ballot_sync(FULL, i < nitems);
        winEnd = __shfl_sync(FULL, wEnd, 31 - __clz(valid));
    };
    load_window(i0);
    for (uint32_t e = e0; e < e1; e += 32 * U) {
        uint32_t ys[U];
        bool ok[U];
        uint64_t src[U][NW];
#pragma unroll
        for (int r = 0; r < U; ++r) {
            const uint32_t er = e + 32 * r;
            ok[r] = false;
            ys[r] = 0;
#pragma unroll
            for (int j = 0; j < NW; ++j) src[r][j] = 0;
            if (er >= e1) continue;  // warp-uniform
            const uint32_t last = min(er + 31, e1 - 1);
            if (last >= winEnd) {
                if (er < winEnd) {
                    const unsigned bal = __ballot_sync(FULL, wE <= er);
                    i0 += 31 - __clz(bal);
                } else {
                    i0 = find_item(Q.eoff, i0, nitems, er);
                }
                load_window(i0);
            }
            const uint32_t ei = er + lane;
            int k = 0;
#pragma unroll
            for (int st = 16; st >= 1; st >>= 1) {
                const uint32_t v = __shfl_sync(FULL, wE, (k + st) & 31);
                if (k + st < 32 && v <= ei) k += st;
            }
            const uint32_t os = __shfl_sync(FULL, wS, k);
            const uint32_t oe = __shfl_sync(FULL, wE, k);
            const int od = __shfl_sync(FULL, wD, k);
#pragma unroll
            for (int j = 0; j < NW; ++j) src[r][j] = __shfl_sync(FULL, w[j], k);
            if (ei < e1) {
                ok[r] = true;
                ys[r] = __ldg((od ? D.adj.dcol : D.adj.col) + os + (ei - oe));
                DBL_DCHECK(ys[r] < D.adj.n);
            }
        }
        uint64_t cur[U][NW];
#pragma unroll
        for (int r = 0; r < U; ++r)
            if (ok[r]) load_words<NW, VEC>(D.lab + (size_t)ys[r] * D.stride, cur[r], D.al);
#pragma unroll
        for (int r = 0; r < U; ++r) {
            if (!ok[r]) continue;
            uint64_t *p = D.lab + (size_t)ys[r] * D.stride;
            bool ch = false;
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                const uint64_t need = src[r][j] & ~cur[r][j];
                if (need) { red_or(p + j, need); ch = true; }
            }
            if (ch) red_or32(D.bits + (ys[r] >> 5), 1u << (ys[r] & 31));
        }
    }
}

// Pull relaxation of the edges [e0, e1) of one adjacency segment (ptr/col):
// row x collects the OR of its neighbours' words over the neighbours that are
// in the current frontier (bitmap cur), with a segmented OR-scan across lanes;
// only a row whose L2-coherent read lacks bits is written (red.or) and marked.
// No per-edge atomics: used for the levels whose frontier covers a large part
// of the graph (direction-optimising, as in push/pull BFS).
template <int NW, bool VEC>
__device__ __forceinline__ void pull_range(const DirParams &D, const uint32_t *__restrict__ ptr,
                                           const uint32_t *__restrict__ col, uint32_t nrows, uint32_t e0,
                                           uint32_t e1) {
    const int lane = threadIdx.x & 31;
    uint32_t x0 = find_item(ptr, 0, nrows, e0);   // ptr[nrows] = m bounds the search
    uint32_t rS = 0xffffffffu, winEnd = 0;
    auto load_window = [&](uint32_t first) {
        const uint32_t i = first + lane;
        rS = i < nrows ? __ldg(ptr + i) : 0xffffffffu;
        const uint32_t last = first + 32 < nrows ? first + 32 : nrows;
        winEnd = __ldg(ptr + last);
    };
    load_window(x0);
    for (uint32_t e = e0; e < e1;) {
        // a 32-row window may hold fewer than 32 edges (empty rows): a round
        // covers the edges of the window only
        if (e >= winEnd) {
            x0 = find_item(ptr, x0, nrows, e);
            load_window(x0);
        } else if (min(e + 31, e1 - 1) >= winEnd) {
            const unsigned bal = __ballot_sync(FULL, rS <= e);
            x0 += 31 - __clz(bal);
            load_window(x0);
        }
        const uint32_t rend = min(min(e + 32, e1), winEnd);
        const uint32_t ei = e + lane;
        const bool ok = ei < rend;
        e = rend;
        int k = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
            const uint32_t v = __shfl_sync(FULL, rS, (k + st) & 31);
            if (k + st < 32 && v <= ei) k += st;
        }
        const uint32_t x = ok ? x0 + k : 0xffffffffu;
        uint64_t acc[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) acc[j] = 0;
        if (ok) {
            const uint32_t p = __ldg(col + ei);
            DBL_DCHECK(p < D.padj.n);
            if ((D.cur[p >> 5] >> (p & 31)) & 1) load_words<NW, VEC>(D.lab + (size_t)p * D.stride, acc, D.al);
        }
        // segmented inclusive OR-scan over lanes holding the same row
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t xo = __shfl_up_sync(FULL, x, o);
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                const uint64_t y = __shfl_up_sync(FULL, acc[j], o);
                if (lane >= o && xo == x) acc[j] |= y;
            }
        }
        const uint32_t xn = __shfl_down_sync(FULL, x, 1);
        const bool seg_last = ok && (lane == 31 || xn != x);
        uint64_t any = 0;
#pragma unroll
        for (int j = 0; j < NW; ++j) any |= acc[j];
        if (seg_last && any) {
            uint64_t *q = D.lab + (size_t)x * D.stride;
            uint64_t cur[NW];
            load_words<NW, VEC>(q, cur, D.al);
            bool ch = false;
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                const uint64_t need = acc[j] & ~cur[j];
                if (need) { red_or(q + j, need); ch = true; }
            }
            if (ch) red_or32(D.bits + (x >> 5), 1u << (x & 31));
        }
    }
}

#if DBL_TRACE
__device__ unsigned long long g_compact_prof[5];   // SM cycles per compaction section, summed over warps
#endif

// Phase B: turn the direction's next-frontier bitmap into the current
// frontier (copied to D.cur) and work items, clearing it.  Each warp owns an
// equal slice of the bitmap; set bits are spread across lanes (32 vertices per
// round) and four rounds are batched so their row-pointer loads are in flight
// together and one 64-bit atomicAdd reserves the slots (and edge offsets) of
// up to 128 vertices.
template <bool COUNT>
__device__ __forceinline__ void compact_bitmap(const DirParams &D, uint32_t nwords, uint32_t gwarp, uint32_t nwarps,
                                               unsigned long long *cnt_ptr, Ctrl *ctrl, uint32_t &nchanged) {
#ifndef DBL_COMPACT_R
#define DBL_COMPACT_R 4
#endif
    constexpr int R = DBL_COMPACT_R;
    const int lane = threadIdx.x & 31;
#if DBL_COMPACT_SLICES
    const uint32_t per = (nwords + nwarps - 1) / nwarps;
    const uint32_t w0 = gwarp * per, w1 = min(w0 + per, nwords), gstep = 32;
#else
    // 32-word groups dealt round-robin over the warps: a frontier whose
    // density varies along the id range (R-MAT leaves gather in the
    // high-id, low-degree part) still gives every warp the same share
    // (contiguous slices: cfg5 level-0 compaction 716 us, mostly warps
    // waiting at the barrier for the densest slices)
    const uint32_t w0 = gwarp * 32, w1 = nwords, gstep = nwarps * 32;
#endif
#if DBL_TRACE
    long long tsec[5] = {0, 0, 0, 0, 0};
    long long tq = clock64();
#define DBL_TSEC(i) do { const long long tn = clock64(); tsec[i] += tn - tq; tq = tn; } while (0)
#else
#define DBL_TSEC(i) do { } while (0)
#endif
    for (uint32_t g0 = w0; g0 < w1; g0 += gstep) {
        const uint32_t wi = g0 + lane;
        const uint32_t bits = wi < w1 ? ld_cg32(D.bits + wi) : 0u;
        if (wi < w1) {
            D.cur[wi] = bits;
            if (bits) D.bits[wi] = 0;
        }
        uint32_t tot = 0;
        const uint32_t excl = warp_excl_scan_u32(__popc(bits), tot);
        DBL_TSEC(0);
        for (uint32_t t0 = 0; t0 < tot; t0 += 32 * R) {
            uint32_t ys[R], b0[R], b1[R], d0[R], d1[R];
            bool val[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t t = t0 + 32 * r + lane;
                int k = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const uint32_t v = __shfl_sync(FULL, excl, (k + st) & 31);
                    if (k + st < 32 && v <= t) k += st;
                }
                const uint32_t ob = __shfl_sync(FULL, bits, k);
                const uint32_t oe = __shfl_sync(FULL, excl, k);
                val[r] = t < tot;
                ys[r] = val[r] ? (g0 + k) * 32 + select_bit(ob, t - oe) : 0u;
            }
            DBL_TSEC(1);
            uint32_t ni = 0, ne = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                b0[r] = b1[r] = d0[r] = d1[r] = 0;
                if (val[r]) {
                    b0[r] = __ldg(D.adj.ptr + ys[r]);
                    b1[r] = __ldg(D.adj.ptr + ys[r] + 1);
                    if (D.adj.dptr) {
                        d0[r] = __ldg(D.adj.dptr + ys[r]);
                        d1[r] = __ldg(D.adj.dptr + ys[r] + 1);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                ni += (b1[r] > b0[r]) + (d1[r] > d0[r]);
                ne += (b1[r] - b0[r]) + (d1[r] - d0[r]);
                if (COUNT && val[r]) {
                    const uint32_t bit = 1u << (ys[r] & 31);
                    const uint32_t old = atomicOr(&D.changed_bits[ys[r] >> 5], bit);
                    if (!(old & bit)) ++nchanged;
                }
            }
            const uint32_t ii = warp_incl_scan(ni), ei = warp_incl_scan(ne);
            DBL_TSEC(2);
            const uint32_t ti = __shfl_sync(FULL, ii, 31), te = __shfl_sync(FULL, ei, 31);
            if (ti == 0) continue;
            unsigned long long base = 0;
            if (lane == 31) base = atomicAdd(cnt_ptr, ((unsigned long long)ti << 32) | te);
            base = __shfl_sync(FULL, base, 31);
            const uint32_t ibase = (uint32_t)(base >> 32), ebase = (uint32_t)base;
            DBL_TSEC(3);
            if ((uint64_t)ibase + ti > D.cap) {
                if (lane == 0) atomicOr(&ctrl->overflow, 1u);
                continue;
            }
            uint32_t pos = ibase + ii - ni, eo = ebase + ei - ne;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (b1[r] > b0[r]) {
                    D.q.x[pos] = ys[r]; D.q.start[pos] = b0[r]; D.q.len[pos] = b1[r] - b0[r]; D.q.eoff[pos] = eo;
                    ++pos;
                    eo += b1[r] - b0[r];
                }
                if (d1[r] > d0[r]) {
                    D.q.x[pos] = ys[r]; D.q.start[pos] = d0[r]; D.q.len[pos] = (d1[r] - d0[r]) | DELTA_BIT;
                    D.q.eoff[pos] = eo;
                    ++pos;
                    eo += d1[r] - d0[r];
                }
            }
            DBL_TSEC(4);
        }
    }
#if DBL_TRACE
    if (lane == 0)
        for (int i = 0; i < 5; ++i) atomicAdd(&g_compact_prof[i], (unsigned long long)tsec[i]);
#endif
#undef DBL_TSEC
}

template <int NW, bool VEC>
__device__ __forceinline__ void relax_part(const DirParams &D, bool pull, uint32_t nitems, uint32_t a, uint32_t b,
                                           uint32_t n, uint32_t mbase) {
    if (!pull) {
        expand_range<NW, VEC>(D, nitems, a, b);
        return;
    }
    // pull space: base segment [0, mbase), then the delta segment
    if (a < mbase) pull_range<NW, VEC>(D, D.padj.ptr, D.padj.col, n, a, b < mbase ? b : mbase);
    if (b > mbase && D.padj.dptr)
        pull_range<NW, VEC>(D, D.padj.dptr, D.padj.dcol, n, a > mbase ? a - mbase : 0u, b - mbase);
}

#ifndef DBL_FMINB
#define DBL_FMINB 4
#endif
template <int NW, bool VEC, bool COUNT>
__global__ void __launch_bounds__(FIX_THREADS, DBL_FMINB) fixpoint_kernel(FixParams P) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nwords = (P.n + 31) / 32;
    Ctrl *ctrl = P.ctrl;
    uint32_t nchanged[2] = {0, 0};
    auto stamp_time = [&](uint32_t slot) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && slot < 64) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            ctrl->level_t[slot] = t;
        }
    };
    for (uint32_t L = 0; L < P.max_levels; ++L) {
        const int cb = L & 1;
        stamp_time(2 * L);
        // phase B: next-frontier bitmaps -> current frontier + work items
        unsigned long long tc0 = 0;
        if (DBL_TRACE && L == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tc0));
#pragma unroll
        for (int d = 0; d < 2; ++d)
            if ((P.active >> d) & 1) compact_bitmap<COUNT>(P.d[d], nwords, warp, nwarps, &ctrl->cnt[cb][d], ctrl, nchanged[d]);
        if (DBL_TRACE && L == 0 && lane == 0) {
            unsigned long long tc1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tc1));
            atomicMax(&ctrl->dbg[0], tc1 - tc0);
            atomicAdd(&ctrl->dbg[1], tc1 - tc0);
            atomicMax(&ctrl->dbg[3], tc0);
        }
        grid.sync();
        const unsigned long long q0 = *(volatile unsigned long long *)&ctrl->cnt[cb][0];
        const unsigned long long q1 = *(volatile unsigned long long *)&ctrl->cnt[cb][1];
        if ((q0 | q1) == 0) {
            if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->levels = L;
            break;
        }
        // phase A: push (edge-balanced over the frontier's items) or pull
        // (edge-balanced over the whole reverse adjacency) per direction
        const uint32_t n0 = (uint32_t)(q0 >> 32), n1 = (uint32_t)(q1 >> 32);
        const uint64_t mall = P.m_base + P.m_delta;
        const bool pull0 = P.pull_div && (uint64_t)(uint32_t)q0 * P.pull_div > mall;
        const bool pull1 = P.pull_div && (uint64_t)(uint32_t)q1 * P.pull_div > mall;
        const uint32_t E0 = pull0 ? (uint32_t)mall : (uint32_t)q0;
        const uint32_t E1 = (q1 == 0) ? 0u : (pull1 ? (uint32_t)mall : (uint32_t)q1);
        const uint32_t E0a = (q0 == 0) ? 0u : E0;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctrl->cnt[cb ^ 1][0] = 0;
            ctrl->cnt[cb ^ 1][1] = 0;
            ctrl->ticket[cb ^ 1] = 0;
            if (L < 32) {
                ctrl->level_edges[L] = (q0 & 0xffffffffull) + (q1 & 0xffffffffull);
                ctrl->level_items[L] = (q0 >> 32) + (q1 >> 32) | ((unsigned long long)(pull0 | (pull1 << 1)) << 60);
            }
        }
        stamp_time(2 * L + 1);
        const uint64_t total = (uint64_t)E0a + E1;
        // dynamic edge tickets: a warp grabs TICKET edges at a time, so slow
        // ranges (hub destinations, L2 misses) do not hold the level back
        // (small levels use a static equal split: the one failing ticket grab
        // per warp would serialise on the counter)
        constexpr uint32_t TICKET = 1024;
        const bool dynamic = total > (uint64_t)nwarps * 512;
        const uint64_t ntick = dynamic ? (total + TICKET - 1) / TICKET : nwarps;
        uint64_t per = (total + nwarps - 1) / nwarps;
        per = (per + 31) & ~31ull;
        for (uint32_t it = 0;; ++it) {
            uint32_t t = 0;
            if (dynamic) {
                if (lane == 0) t = atomicAdd(&ctrl->ticket[cb], 1u);
                t = __shfl_sync(FULL, t, 0);
            } else {
                t = it == 0 ? warp : 0xffffffffu;
            }
            if (t >= ntick) break;
            const uint64_t sz = dynamic ? TICKET : per;
            const uint64_t a = (uint64_t)t * sz, b = (a + sz < total) ? a + sz : total;
            if (a >= b) break;
            if (a < E0a)
                relax_part<NW, VEC>(P.d[0], pull0, n0, (uint32_t)a, (uint32_t)(b < E0a ? b : (uint64_t)E0a), P.n,
                                    (uint32_t)P.m_base);
            if (b > E0a)
                relax_part<NW, VEC>(P.d[1], pull1, n1, a > E0a ? (uint32_t)(a - E0a) : 0u, (uint32_t)(b - E0a), P.n,
                                    (uint32_t)P.m_base);
        }
        grid.sync();
    }
    if (COUNT) {
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            uint32_t v = nchanged[d];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
            if (lane == 0 && v) atomicAdd(&ctrl->changed[d], (unsigned long long)v);
        }
    }
}

// ------------------------------------------------------- seeds & frontier --

// rec := seeds, one thread per vertex writing its whole record (16-byte
// stores when every word is selected).  bl_in bit bucket[v] for source
// leaves, bl_out for sinks; dl words zero (landmark bits are added by
// landmark_bits_kernel).
__global__ void seed_records_kernel(uint64_t *__restrict__ rec, uint32_t n, uint32_t wdl, uint32_t wbl,
                                    const uint8_t *__restrict__ flags, const uint32_t *__restrict__ bucket,
                                    uint64_t wmask) {
    const uint32_t H = wdl + wbl, rw = 2 * H, rs = rec_stride(H);
    const bool all = (rw >= 64) ? wmask == ~0ull : (wmask & ((1ull << rw) - 1)) == ((1ull << rw) - 1);
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint8_t f = flags[v];
        const uint32_t b = bucket[v];
        uint64_t *r = rec + (size_t)v * rs;
        // word index of the bucket bit in each half (or none)
        const uint32_t win = (f & 1) ? wdl + b / 64 : 0xffffffffu;
        const uint32_t wout = (f & 2) ? H + wdl + b / 64 : 0xffffffffu;
        const uint64_t bit = 1ull << (b % 64);
        for (uint32_t w = rw; w < rs; ++w) r[w] = 0ull;   // pad words
        if (all) {
            for (uint32_t w = 0; w < rw; w += 2) {
                ulonglong2 val;
                val.x = (w == win || w == wout) ? bit : 0ull;
                val.y = (w + 1 == win || w + 1 == wout) ? bit : 0ull;
                *reinterpret_cast<ulonglong2 *>(r + w) = val;
            }
        } else {
            for (uint32_t w = 0; w < rw; ++w)
                if ((wmask >> w) & 1) r[w] = (w == win || w == wout) ? bit : 0ull;
        }
    }
}

__global__ void landmark_bits_kernel(uint64_t *__restrict__ rec, uint32_t rs, uint32_t H,
                                     const uint32_t *__restrict__ lm, uint32_t k, uint64_t wmask) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        const uint64_t v = lm[i];
        if ((wmask >> (i / 64)) & 1)
            atomicOr(reinterpret_cast<unsigned long long *>(rec + v * rs + i / 64), 1ull << (i % 64));
        if ((wmask >> (H + i / 64)) & 1)
            atomicOr(reinterpret_cast<unsigned long long *>(rec + v * rs + H + i / 64), 1ull << (i % 64));
    }
}

// Level-0 frontier bitmaps straight from the metadata: vertex v starts
// direction d's frontier iff it seeds one of the words [w0_d, w0_d + nw_d) of
// that half -- a leaf of side d whose bucket word is in range, or a landmark
// whose DL word is (landmark_frontier_kernel).  One ballot per 32 vertices.
__global__ void leaf_frontier_kernel(uint32_t *__restrict__ bits0, uint32_t *__restrict__ bits1, uint32_t n,
                                     uint32_t wdl, uint32_t H, const uint8_t *__restrict__ flags,
                                     const uint32_t *__restrict__ bucket, uint32_t a0, uint32_t e0, uint32_t a1,
                                     uint32_t e1, const Adj fwd, const Adj rev) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t nr = ((uint64_t)n + 31) & ~31ull;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nr; i += stride) {
        bool p0 = false, p1 = false;
        if (i < n) {
            const uint8_t f = flags[i];
            if (f) {
                const uint32_t bw = wdl + bucket[i] / 64;
                p0 = (f & 1) && bw >= a0 && bw < e0;
                p1 = (f & 2) && H + bw >= a1 && H + bw < e1;
                // only with edges to push along (as in prep_kernel)
                if (p0) p0 = fwd.ptr[i + 1] > fwd.ptr[i] || (fwd.dptr && fwd.dptr[i + 1] > fwd.dptr[i]);
                if (p1) p1 = rev.ptr[i + 1] > rev.ptr[i] || (rev.dptr && rev.dptr[i + 1] > rev.dptr[i]);
            }
        }
        const unsigned b0 = __ballot_sync(FULL, p0), b1 = __ballot_sync(FULL, p1);
        if ((threadIdx.x & 31) == 0) {
            if (bits0) bits0[i >> 5] = b0;
            if (bits1) bits1[i >> 5] = b1;
        }
    }
}

__global__ void landmark_frontier_kernel(uint32_t *__restrict__ bits0, uint32_t *__restrict__ bits1, uint32_t H,
                                         const uint32_t *__restrict__ lm, uint32_t k, uint32_t a0, uint32_t e0,
                                         uint32_t a1, uint32_t e1) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        const uint32_t v = lm[i], w = i / 64;
        if (bits0 && w >= a0 && w < e0) atomicOr(&bits0[v >> 5], 1u << (v & 31));
        if (bits1 && H + w >= a1 && H + w < e1) atomicOr(&bits1[v >> 5], 1u << (v & 31));
    }
}

// Insertion seeds (updates.py:129-134 for a whole batch): for each new edge
// u->v, in-words(v) |= in-words(u) and out-words(u) |= out-words(v); changed
// endpoints start the level-0 frontier.
template <int NW, bool VEC>
__global__ void insert_seed_kernel(FixParams P, const uint64_t *__restrict__ keys, uint64_t count,
                                   const uint64_t *__restrict__ count_dev) {
    if (count_dev) count = *count_dev;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        const uint32_t u = (uint32_t)(key >> 32), v = (uint32_t)key;
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            const DirParams &D = P.d[d];
            const uint32_t src = d == 0 ? u : v, dst = d == 0 ? v : u;
            uint64_t s[NW];
            load_words<NW, VEC>(D.lab + (size_t)src * D.stride, s, D.al);
            if (relax_mark<NW, VEC>(D, dst, s)) atomicOr(&P.ctrl->seed_changed[d], 1u);
        }
    }
}

// ------------------------------------------------------------ host driver --

struct Group { int dir; uint32_t w0, nw; };

static void plan_groups(const dbl_index *idx, const uint32_t *words, uint32_t nwords,
                        Group *out, int &ng) {
    // words of each half, in order; split into runs of contiguous words of
    // <= MAX_GROUP_WORDS each.
    const uint32_t H = idx->wdl + idx->wbl;
    ng = 0;
    for (int d = 0; d < 2; ++d) {
        bool sel[2 * MAX_SHARD_WORDS + 2] = {};
        uint32_t cnt = 0;
        for (uint32_t w = 0; w < H; ++w) {
            bool s = true;
            if (words) {
                s = false;
                for (uint32_t i = 0; i < nwords; ++i) if (words[i] == d * H + w) s = true;
            }
            sel[w] = s;
            cnt += s;
        }
        (void)cnt;
        uint32_t w = 0;
        while (w < H) {
            if (!sel[w]) { ++w; continue; }
            uint32_t e = w;
            while (e < H && sel[e] && e - w < (uint32_t)MAX_GROUP_WORDS) ++e;
            out[ng++] = Group{d, d * H + w, e - w};
            w = e;
        }
    }
}

template <int NW, bool VEC, bool COUNT>
static dbl_status launch_fixpoint_t(dbl_graph *g, FixParams &P) {
    auto kern = fixpoint_kernel<NW, VEC, COUNT>;
    int blocks_per_sm = 1;
    dbl_status s = kernel_occupancy((const void *)kern, FIX_THREADS, 0, &blocks_per_sm);
    if (s) return s;
    // CTAs per SM: the occupancy maximum for builds; insert runs (COUNT)
    // use 2 (grid barriers get cheaper with fewer CTAs and insert levels
    // are small: 100k-edge batches 0.54 -> 0.52 ms)
    const int cap = COUNT ? DBL_FIX_BPS_INSERT : DBL_FIX_BPS_BUILD;
    const int bps = (cap > 0 && cap < blocks_per_sm) ? cap : blocks_per_sm;
    int grid = bps * g->sm_count;
    void *args[] = {(void *)&P};
    DBL_CUDA(cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(FIX_THREADS), args, 0,
                                         g->stream));
    DBL_LAUNCHED();
    return DBL_OK;
}

template <bool COUNT>
static dbl_status launch_fixpoint(dbl_graph *g, FixParams &P, uint32_t nw, bool vec) {
#define DBL_FIX_CASE(N)                                                            \
    case N:                                                                        \
        return vec ? launch_fixpoint_t<N, (N % 2 == 0), COUNT>(g, P)               \
                   : launch_fixpoint_t<N, false, COUNT>(g, P);
    switch (nw) {
        DBL_FIX_CASE(1) DBL_FIX_CASE(2) DBL_FIX_CASE(3) DBL_FIX_CASE(4)
        DBL_FIX_CASE(5) DBL_FIX_CASE(6) DBL_FIX_CASE(7) DBL_FIX_CASE(8)
    default: set_error("bad word-group width"); return DBL_E_CONFIG;
    }
#undef DBL_FIX_CASE
}

static dbl_status launch_init_frontier(dbl_graph *g, dbl_index *idx, const Group *pair[2]) {
    const uint32_t H = idx->wdl + idx->wbl;
    uint32_t *b0 = pair[0] ? g->stamp[0].as<uint32_t>() : nullptr;
    uint32_t *b1 = pair[1] ? g->stamp[1].as<uint32_t>() : nullptr;
    const uint32_t a0 = pair[0] ? pair[0]->w0 : 0, e0 = pair[0] ? pair[0]->w0 + pair[0]->nw : 0;
    const uint32_t a1 = pair[1] ? pair[1]->w0 : 0, e1 = pair[1] ? pair[1]->w0 + pair[1]->nw : 0;
    int blocks = (int)(((uint64_t)g->n + 255) / 256);
    if (blocks > g->sm_count * 8) blocks = g->sm_count * 8;
    if (blocks < 1) blocks = 1;
    leaf_frontier_kernel<<<blocks, 256, 0, g->stream>>>(b0, b1, g->n, idx->wdl, H, idx->leaf_flags.as<uint8_t>(),
                                                         idx->bucket.as<uint32_t>(), a0, e0, a1, e1, graph_fwd(g),
                                                         graph_rev(g));
    DBL_CHECK_LAUNCH("leaf_frontier_kernel");
    if (idx->cfg.k) {
        landmark_frontier_kernel<<<(idx->cfg.k + 255) / 256, 256, 0, g->stream>>>(
            b0, b1, H, idx->landmarks.as<uint32_t>(), idx->cfg.k, a0, e0, a1, e1);
        DBL_CHECK_LAUNCH("landmark_frontier_kernel");
    }
    return DBL_OK;
}

static dbl_status launch_insert_seed(dbl_graph *g, FixParams &P, uint32_t nw, bool vec, bool /*count*/,
                                     const uint64_t *keys, uint64_t nk, const uint64_t *nk_dev) {
    int blocks = (int)((nk + 255) / 256);
    if (blocks > g->sm_count * 8) blocks = g->sm_count * 8;
    if (blocks < 1) blocks = 1;
#define DBL_SEED_CASE(N)                                                                      \
    case N:                                                                                   \
        if (vec) insert_seed_kernel<N, (N % 2 == 0)><<<blocks, 256, 0, g->stream>>>(P, keys, nk, nk_dev); \
        else insert_seed_kernel<N, false><<<blocks, 256, 0, g->stream>>>(P, keys, nk, nk_dev);       \
        break;
    switch (nw) {
        DBL_SEED_CASE(1) DBL_SEED_CASE(2) DBL_SEED_CASE(3) DBL_SEED_CASE(4)
        DBL_SEED_CASE(5) DBL_SEED_CASE(6) DBL_SEED_CASE(7) DBL_SEED_CASE(8)
    default: set_error("bad word-group width"); return DBL_E_CONFIG;
    }
#undef DBL_SEED_CASE
    DBL_CHECK_LAUNCH("insert_seed_kernel");
    return DBL_OK;
}

static dbl_status prepare_params(dbl_graph *g, dbl_index *idx, const Group *gr[2], FixParams &P,
                                 uint32_t &nw, bool &vec, bool count, bool reset_counts = true,
                                 bool clear_bits = true) {
    dbl_status s = graph_ensure_traversal(g);
    if (s) return s;
    const size_t bmw = ((size_t)g->n + 31) / 32;
    if (clear_bits) {
        DBL_CUDA(cudaMemsetAsync(g->stamp[0].p, 0, bmw * 4, g->stream));
        DBL_CUDA(cudaMemsetAsync(g->stamp[1].p, 0, bmw * 4, g->stream));
    }
    nw = 0;
    vec = true;
    for (int d = 0; d < 2; ++d) {
        DirParams &D = P.d[d];
        D.adj = d == 0 ? graph_fwd(g) : graph_rev(g);
        D.padj = d == 0 ? graph_rev(g) : graph_fwd(g);
        D.stride = idx->rs;
        D.bits = g->stamp[d].as<uint32_t>();
        D.cur = D.bits + bmw + 1;
        D.cap = g->qcap;
        {
            uint32_t *b = g->qbuf[d][0].as<uint32_t>();
            D.q.x = b;
            D.q.start = b + g->qcap;
            D.q.len = b + 2ull * g->qcap;
            D.q.eoff = b + 3ull * g->qcap;
        }
        D.changed_bits = count ? g->changed_bits.as<uint32_t>() + d * (((size_t)g->n + 31) / 32) : nullptr;
        if (gr[d]) {
            D.lab = idx->rec.as<uint64_t>() + gr[d]->w0;
            D.al = (idx->rs % 4 == 0) ? (int)(gr[d]->w0 % 4) : -1;
            nw = gr[d]->nw;
            if ((gr[d]->w0 % 2) || (idx->rs % 2)) vec = false;
        } else {
            D.lab = idx->rec.as<uint64_t>();
            D.al = -1;
        }
    }
    P.ctrl = g->ctrl.as<Ctrl>();
    P.m_base = g->m_base;
    P.m_delta = g->m_delta;
    // pull measured slower than push on cfg2 (r01): off unless a variant
    // build asks for it (-DDBL_PULL_DIV=d)
    P.pull_div = DBL_PULL_DIV;   // 0 disables pull
    P.n = g->n;
    P.active = (gr[0] ? 1u : 0u) | (gr[1] ? 2u : 0u);
    P.max_levels = g->n + 4;
    DBL_CUDA(cudaMemsetAsync(P.ctrl, 0, sizeof(Ctrl), g->stream));
    if (count && reset_counts)
        DBL_CUDA(cudaMemsetAsync(g->changed_bits.p, 0, (((size_t)g->n + 31) / 32) * 2 * 4, g->stream));
    return DBL_OK;
}

// Read the run's control block (and, for the first run of a build, the prep
// state) through pinned staging with ONE stream synchronisation; the ev[1]
// timestamp of the run is recorded before it.
static dbl_status finish_run(dbl_graph *g, Ctrl *hctrl, PrepState *hprep = nullptr,
                             const unsigned long long *extra_dev = nullptr, unsigned long long *extra_host = nullptr) {
    dbl_status s = g->host_stage.ensure(sizeof(Ctrl) + sizeof(PrepState) + 128);
    if (s) return s;
    Ctrl *pc = reinterpret_cast<Ctrl *>(g->host_stage.p);
    PrepState *pp = reinterpret_cast<PrepState *>(reinterpret_cast<char *>(g->host_stage.p) +
                                                  ((sizeof(Ctrl) + 15) & ~size_t(15)));
    DBL_CUDA(cudaMemcpyAsync(pc, g->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, g->stream));
    if (hprep) DBL_CUDA(cudaMemcpyAsync(pp, g->prep.p, sizeof(PrepState), cudaMemcpyDeviceToHost, g->stream));
    unsigned long long *pe = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(pp) +
                                                                    ((sizeof(PrepState) + 15) & ~size_t(15)));
    if (extra_dev) DBL_CUDA(cudaMemcpyAsync(pe, extra_dev, 32, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaEventRecord(g->ev[1], g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    *hctrl = *pc;
    if (hprep) *hprep = *pp;
    if (extra_dev)
        for (int k = 0; k < 4; ++k) extra_host[k] = pe[k];
    if (hctrl->overflow) { set_error("frontier queue overflow"); return DBL_E_CUDA; }
    return DBL_OK;
}

dbl_status index_seed_records(dbl_graph *g, dbl_index *idx, uint64_t wmask) {
    const uint64_t total = (uint64_t)idx->n * idx->rw;
    if (!total) return DBL_OK;
    int blocks = (int)((idx->n + 255) / 256 < (uint32_t)g->sm_count * 8 ? (idx->n + 255) / 256 : g->sm_count * 8);
    seed_records_kernel<<<blocks, 256, 0, g->stream>>>(idx->rec.as<uint64_t>(), idx->n, idx->wdl, idx->wbl,
                                                       idx->leaf_flags.as<uint8_t>(), idx->bucket.as<uint32_t>(),
                                                       wmask);
    DBL_CHECK_LAUNCH("seed_records_kernel");
    if (idx->cfg.k) {
        landmark_bits_kernel<<<(idx->cfg.k + 255) / 256, 256, 0, g->stream>>>(
            idx->rec.as<uint64_t>(), idx->rs, idx->wdl + idx->wbl, idx->landmarks.as<uint32_t>(), idx->cfg.k,
            wmask);
        DBL_CHECK_LAUNCH("landmark_bits_kernel");
    }
    return DBL_OK;
}

// ------------------------------------------------------ pivot head start --
//
// Labels are least fixpoints, so any vertex may start from any subset of its
// final label without changing the result.  Pick a pivot h (landmark 0, the
// top-ranked hub) and compute D(h) = vertices reachable from h and A(h) =
// vertices reaching h with a one-bit fixpoint per direction.  Every x in
// D(h) ends with L_in(x) >= L_in(h) = OR of the in-seeds over A(h), every
// x in A(h) with L_out(x) >= L_out(h) = OR of the out-seeds over D(h), so
// those unions are ORed in before the label fixpoint.  D(h) is closed under
// successors and A(h) under predecessors, so the head-start bits need no
// propagation of their own: the label fixpoint then only moves the seed bits
// the pivot's unions do not already hold.  On R-MAT the pivot's SCC holds
// every seed bit, so this replaces the two label levels that relax almost
// every edge (with multi-bit labels) by one single-bit reachability sweep
// per direction.

// Reachability of the pivot by bottom-up sweeps (direction-optimised BFS
// without the top-down levels after the first): vis[0] = reached from h,
// vis[1] = reaches h.  Each sweep, every unmarked vertex scans its
// predecessors in that direction (in-edges for vis[0], out-edges for vis[1])
// and stops at the first marked one -- on R-MAT almost every vertex of the
// giant SCC finds a marked hub among its first neighbours, so a sweep costs
// about one neighbour check per vertex instead of a push along every edge.
// Marks made during a sweep may be seen by later vertices of the same sweep
// (fewer sweeps); a stale L1 copy only defers a mark to the next sweep.
struct ReachParams {
    uint64_t *rec;       // records (seeded): unions over A(h)/D(h) are ORed in at the end
    unsigned long long *L;   // 2H words of unions
    uint64_t wmask;          // record words being built (bit w = word w)
    uint64_t cap_wmask;      // words whose level-0 frontier is `front` (used when the sweeps are capped)
    uint32_t *front[2];      // level-0 frontier bitmaps of the label fixpoint (or nullptr)
    uint32_t *dmask_out;     // copy of vis[0] kept with the index (or nullptr)
    unsigned long long *scc_out;   // DL bits of the landmarks in h's SCC (wdl words)
    uint32_t k, wdl;
    uint32_t H;
    Adj adj[2];          // [0] in-edges (reverse adjacency), [1] out-edges (forward adjacency)
    Adj top[2];          // first level from h: [0] out-edges, [1] in-edges
    uint32_t *vis[2];
    uint32_t *nb[2][3];      // per direction: vertices newly marked in step s go to nb[d][s % 3]
    unsigned int *changed;   // [step % 3]: marks made in step s (read after its barrier, cleared in s + 2);
                             // [3]: set when the step cap stopped the search (no head start then);
                             // [4]: steps run, [5]: bottom-up sweeps among them (trace);
                             // [6]: apply CTAs done
    uint32_t max_sweeps;     // cap on bottom-up sweeps (each O(n))
    uint32_t max_steps;      // cap on all steps
    uint32_t td_switch;      // switch to top-down once a step marks fewer vertices than this
    unsigned long long *tr;  // trace (or nullptr): [2s] end time of step s (globaltimer), [2s+1] its marks
    unsigned long long *work;   // executed work (dbl_build_work_stats): [0] bottom-up vertex tests, [1] their
                                // neighbour probes, [2] top-down frontier vertices, [3] their edges,
                                // [4] records the union pass touched
    const uint32_t *lm;
    const uint8_t *flags;    // leaf flags and buckets: the seeds, read instead of the seeded records
    const uint32_t *bucket;
    bool write_rec;          // records not seeded yet (full build): write seeds | head start, whole lines
    uint32_t n, nwords;
    uint32_t kp;             // k_prime (bucket bits per BL half)
    const uint32_t *haspred[2];   // vertices with a predecessor along adj[d] (prep), or nullptr
    uint32_t sparse_g;            // bitmap words per warp step in the sparse sweeps (power of 2, <= 32)
    bool fused_apply;        // apply the head start inside reach_kernel (small graphs)
};

__device__ __forceinline__ bool vis_test_ca(const uint32_t *vis, uint32_t x) {
    uint32_t w;
    asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(w) : "l"(vis + (x >> 5)));
    return (w >> (x & 31)) & 1u;
}

__device__ __forceinline__ bool any_marked(const Adj &a, const uint32_t *vis, uint32_t x) {
    // one neighbour at a time: most vertices stop at their first or second
    // neighbour, and batching 4 or 8 loads per step measured slower (cfg2
    // first sweep 40 -> 60 us, cfg5 1.4 -> 3.3 ms)
    uint32_t s0 = __ldg(a.ptr + x), s1 = __ldg(a.ptr + x + 1);
    for (uint32_t j = s0; j < s1; ++j)
        if (vis_test_ca(vis, __ldg(a.col + j))) return true;
    if (a.dptr) {
        s0 = __ldg(a.dptr + x);
        s1 = __ldg(a.dptr + x + 1);
        for (uint32_t j = s0; j < s1; ++j)
            if (vis_test_ca(vis, __ldg(a.dcol + j))) return true;
    }
    return false;
}

// CTAs per SM as a template: 6 (40 registers, no spills) is best on cfg2
// (8: 0.283, 6: 0.280, 4: 0.287 ms per build), 8 (32 registers, a few spills)
// on cfg5's 2^26 vertices (reach 4.8 vs 5.1 ms): the latency-bound sweeps
// want the occupancy once the graph is large
#ifndef DBL_BU_ILP
#define DBL_BU_ILP 1
#endif
// The head start into the records (after the unions): vertices of h's SCC
// leave the level-0 frontier, then every record takes L_in(h) / L_out(h) by
// membership (and, in write mode, its seeds).  FAST adds the write-mode path
// for strides dividing 64 words (more registers: used by the stand-alone
// apply kernel; the fused small-graph variant inside reach_kernel keeps the
// general loop and the sweeps' register budget).
template <bool WORK, int FAST>
__device__ __forceinline__ void apply_head_start(const ReachParams &P, uint64_t tid, uint64_t nth,
                                                 const unsigned long long *acc, bool drop, bool capped) {
    const uint32_t H = P.H, rw = 2 * H, rs = rec_stride(H);
    // a vertex of h's SCC (in D(h) and A(h)) now holds L_in(h) / L_out(h),
    // which every successor / predecessor also holds: it leaves the level-0
    // frontier (on R-MAT that drops the landmarks, the hubs of that frontier)
    for (uint64_t w = tid; w < P.nwords && !drop; w += nth) {
        if (capped) {   // partial sets: every marked vertex propagates its head start
            P.front[0][w] |= P.vis[0][w];
            P.front[1][w] |= P.vis[1][w];
            continue;
        }
        const uint32_t scc = P.vis[0][w] & P.vis[1][w];
        if (scc) {
            if (P.front[0]) P.front[0][w] &= ~scc;
            if (P.front[1]) P.front[1][w] &= ~scc;
        }
    }
    // apply: a warp takes 32 consecutive records (one bitmap word per
    // direction) and ORs the unions in with 512-byte coalesced
    // read-modify-writes, instead of 8-byte accesses at the record stride.
    // In write mode (full build, prep skipped the records) it writes every
    // record whole instead -- seeds from the metadata | the unions, pad words
    // zero -- with no read at all, and the landmark bits follow.
    {
        const int lane = threadIdx.x & 31;
        const uint32_t wdl = P.wdl;
        const uint64_t nblk = P.nwords, gw = tid >> 5, nw = nth >> 5;
        unsigned long long touched = 0;
        // lane's first (record, word) in a block and the step per 64 words,
        // so the store loop needs no division by the runtime stride
        const uint32_t r0 = (2 * lane) / rs, w0 = (2 * lane) % rs, q64 = 64 / rs, m64 = 64 % rs;
        if (FAST == 2 && P.write_rec) {
            // write mode, stride dividing 128 words (k <= 960 at k' = 64):
            // 32-byte stores (a warp instruction covers 1 KB, 128 / rs
            // records); a lane's 4 words w..w+3 are the same in every store,
            // so its union words are fixed; the next block's bitmap words,
            // flags and buckets load while this block's records are stored
            const uint32_t w = (4 * lane) % rs, rq0 = (4 * lane) / rs, q = 128 / rs;
            // a 32-byte sector holding only pad words is not written (pads
            // are unspecified; readers use words < 2H): at k = 256 the
            // 128-byte records are written as 96 bytes, a quarter less traffic
            const bool live = w < 2 * H;
            uint64_t Aw[4];
            bool hw[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                Aw[j] = w + j < rw ? acc[w + j] : 0ull;
                hw[j] = w + j < H;
            }
            uint32_t fb = 0, bb = 0, f = 0, b = 0;
            auto fetch = [&](uint64_t blk) {
                fb = drop ? 0u : P.vis[0][blk];
                bb = drop ? 0u : P.vis[1][blk];
                const uint64_t v = blk * 32 + lane;
                f = v < P.n ? P.flags[v] : 0u;
                b = v < P.n ? P.bucket[v] : 0u;
            };
            if (gw < nblk) fetch(gw);
            for (uint64_t blk = gw; blk < nblk; blk += nw) {
                const uint32_t cfb = fb, cbb = bb, cf = f, cbk = b;
                if (blk + nw < nblk) fetch(blk + nw);
                if (WORK && lane == 0) touched += __popc(cfb | cbb);
                const uint32_t sb = cbk % 64;
                const uint32_t win = (cf & 1) ? wdl + cbk / 64 : 0xffffffffu;
                const uint32_t wout = (cf & 2) ? H + wdl + cbk / 64 : 0xffffffffu;
                uint64_t *base = P.rec + blk * 32 * rs;
                uint32_t r = rq0;
                for (uint32_t t = 0; t < rs * 32; t += 128, r += q) {
                    const uint32_t swin = __shfl_sync(FULL, win, r), swout = __shfl_sync(FULL, wout, r);
                    const uint64_t sbit = 1ull << __shfl_sync(FULL, sb, r);
                    const bool in_d = (cfb >> r) & 1u, in_a = (cbb >> r) & 1u;
                    if (!live || blk * 32 + r >= P.n) continue;
                    uint64_t val[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        val[j] = ((hw[j] ? in_d : in_a) ? Aw[j] : 0ull) |
                                 ((w + j == swin || w + j == swout) ? sbit : 0ull);
                    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(base + t + 4 * lane), "l"(val[0]),
                                 "l"(val[1]), "l"(val[2]), "l"(val[3])
                                 : "memory");
                }
            }
        } else if (FAST == 1 && P.write_rec && m64 == 0) {
            // write mode, stride dividing 64 words (every stride up to
            // k = 448): a lane's word pair w0 is the same in every store, so
            // its union words are fixed; the next block's bitmap words, flags
            // and buckets load while this block's records are stored
            const uint32_t w = w0;
            const uint64_t A0 = w < rw ? acc[w] : 0ull, A1 = w + 1 < rw ? acc[w + 1] : 0ull;
            const bool h0 = w < H, h1 = w + 1 < H;
            uint32_t fb = 0, bb = 0, f = 0, b = 0;
            auto fetch = [&](uint64_t blk) {
                fb = drop ? 0u : P.vis[0][blk];
                bb = drop ? 0u : P.vis[1][blk];
                const uint64_t v = blk * 32 + lane;
                f = v < P.n ? P.flags[v] : 0u;
                b = v < P.n ? P.bucket[v] : 0u;
            };
            if (gw < nblk) fetch(gw);
            for (uint64_t blk = gw; blk < nblk; blk += nw) {
                const uint32_t cfb = fb, cbb = bb, cf = f, cbk = b;
                if (blk + nw < nblk) fetch(blk + nw);
                if (WORK && lane == 0) touched += __popc(cfb | cbb);
                const uint32_t sb = cbk % 64;
                const uint32_t win = (cf & 1) ? wdl + cbk / 64 : 0xffffffffu;
                const uint32_t wout = (cf & 2) ? H + wdl + cbk / 64 : 0xffffffffu;
                uint64_t *base = P.rec + blk * 32 * rs;
                uint32_t r = r0;
                for (uint32_t t = 0; t < rs * 32; t += 64, r += q64) {
                    const uint32_t swin = __shfl_sync(FULL, win, r), swout = __shfl_sync(FULL, wout, r);
                    const uint64_t sbit = 1ull << __shfl_sync(FULL, sb, r);
                    const bool in_d = (cfb >> r) & 1u, in_a = (cbb >> r) & 1u;
                    if (blk * 32 + r >= P.n) continue;
                    ulonglong2 val;
                    val.x = ((h0 ? in_d : in_a) ? A0 : 0ull) | ((w == swin || w == swout) ? sbit : 0ull);
                    val.y = ((h1 ? in_d : in_a) ? A1 : 0ull) | ((w + 1 == swin || w + 1 == swout) ? sbit : 0ull);
                    *reinterpret_cast<ulonglong2 *>(base + t + 2 * lane) = val;
                }
            }
        } else
        for (uint64_t blk = gw; blk < nblk; blk += nw) {
            const uint32_t fb = drop ? 0u : P.vis[0][blk], bb = drop ? 0u : P.vis[1][blk];
            if (WORK && lane == 0) touched += __popc(fb | bb);
            if (!(fb | bb) && !P.write_rec) continue;
            uint64_t *base = P.rec + blk * 32 * rs;
            uint32_t win = 0xffffffffu, wout = 0xffffffffu, sb = 0;
            if (P.write_rec) {
                const uint64_t v = blk * 32 + lane;
                if (v < P.n) {
                    const uint8_t f = P.flags[v];
                    if (f) {
                        const uint32_t b = P.bucket[v];
                        sb = b % 64;
                        if (f & 1) win = wdl + b / 64;
                        if (f & 2) wout = H + wdl + b / 64;
                    }
                }
            }
            uint32_t r = r0, w = w0;
            for (uint32_t t = 0; t < rs * 32; t += 64, r += q64, w += m64) {
                if (w >= rs) { w -= rs; ++r; }
                const uint32_t wi = t + 2 * lane;
                const bool in_d = (fb >> r) & 1u, in_a = (bb >> r) & 1u;
                const uint64_t a0 = (w < H ? in_d : (w < rw && in_a)) ? acc[w] : 0ull;
                const uint64_t a1 = (w + 1 < H ? in_d : (w + 1 < rw && in_a)) ? acc[w + 1] : 0ull;
                if (P.write_rec) {
                    const uint32_t swin = __shfl_sync(FULL, win, r), swout = __shfl_sync(FULL, wout, r);
                    const uint64_t sbit = 1ull << __shfl_sync(FULL, sb, r);
                    if (blk * 32 + r >= P.n) continue;
                    ulonglong2 val;
                    val.x = a0 | ((w == swin || w == swout) ? sbit : 0ull);
                    val.y = a1 | ((w + 1 == swin || w + 1 == swout) ? sbit : 0ull);
                    *reinterpret_cast<ulonglong2 *>(base + wi) = val;
                } else if (a0 | a1) {
                    if (blk * 32 + r >= P.n) continue;
                    ulonglong2 *p = reinterpret_cast<ulonglong2 *>(base + wi);
                    ulonglong2 val = *p;
                    val.x |= a0;
                    val.y |= a1;
                    *p = val;
                }
            }
        }
        if (WORK && lane == 0 && touched) atomicAdd(&P.work[4], touched);
    }
}

template <int MINB, bool WORK>
__global__ void __launch_bounds__(256, MINB) reach_kernel(ReachParams P) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t h = P.lm[0];
    const bool have = h < P.n;   // grid-uniform (landmarks are validated, so always in practice)
    if (!have && !P.write_rec) return;   // no pivot, no head start
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    // h and its direct successors / predecessors (top-down first level)
    if (have && tid == 0) {
        atomicOr(&P.vis[0][h >> 5], 1u << (h & 31));
        atomicOr(&P.vis[1][h >> 5], 1u << (h & 31));
    }
#pragma unroll
    for (int d = 0; d < 2 && have; ++d) {
        const Adj &a = P.top[d];
        const uint32_t s0 = a.ptr[h], s1 = a.ptr[h + 1];
        for (uint64_t j = s0 + tid; j < s1; j += nth) {
            const uint32_t y = a.col[j];
            DBL_DCHECK(y < P.n);
            atomicOr(&P.vis[d][y >> 5], 1u << (y & 31));
        }
        if (a.dptr) {
            const uint32_t t0 = a.dptr[h], t1 = a.dptr[h + 1];
            for (uint64_t j = t0 + tid; j < t1; j += nth) {
                const uint32_t y = a.dcol[j];
                DBL_DCHECK(y < P.n);
                atomicOr(&P.vis[d][y >> 5], 1u << (y & 31));
            }
        }
    }
    grid.sync();
    if (P.tr && tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.tr[64] = t;
    }
    // Steps: bottom-up sweeps while they mark many vertices, then top-down
    // levels from the vertices the previous step marked (a bottom-up sweep
    // rescans every unmarked vertex's edges, which in the tail is mostly the
    // vertices outside D(h)/A(h); a top-down level only touches the out-edges
    // of the few new marks).  Every mark is also recorded in nb[d][s % 3].
    bool capped = false, td = false;
    uint32_t bu = 0;
    unsigned prev_got = 0xffffffffu;
    uint32_t w_tests = 0, w_probes = 0, w_tdv = 0, w_tde = 0;   // per-thread work counts
    for (uint32_t step = 0; have; ++step) {
        if (step == P.max_steps || (!td && bu == P.max_sweeps)) {
            // deep graph: the marked sets are only parts of D(h) / A(h), not
            // closed under successors / predecessors.  The head start is
            // still a subset of every marked vertex's final label, so it is
            // kept when the marked vertices can join the level-0 frontier
            // (they then propagate it), and dropped otherwise.
            capped = true;
            if (tid == 0) { P.changed[3] = 1; P.changed[4] = step; P.changed[5] = bu; }
            break;
        }
        const int cb = step % 3;
        unsigned marks = 0;
        if (!td && bu > 0 && P.haspred[0]) {
            // later bottom-up sweeps: only the vertices still unmarked that
            // have a predecessor at all (cfg2 after the first sweep: ~170k of
            // the 1.3M unmarked vertex-directions), picked from the bitmaps
            // 32 words per warp step and spread over the lanes
            const int lane = threadIdx.x & 31;
#pragma unroll 1
            for (int d = 0; d < 2; ++d) {
                const Adj &a = P.adj[d];
                // G words per warp step (host: enough groups for every warp)
                const uint32_t G = P.sparse_g;
                for (uint64_t g0 = (tid >> 5) * G; g0 < P.nwords; g0 += (nth >> 5) * G) {
                    const uint64_t wi = g0 + lane;
                    const uint32_t cand =
                        lane < G && wi < P.nwords ? ~*(volatile uint32_t *)&P.vis[d][wi] & P.haspred[d][wi] : 0u;
                    uint32_t tot = 0;
                    const uint32_t excl = warp_excl_scan_u32(__popc(cand), tot);
                    for (uint32_t t0 = 0; t0 < tot; t0 += 32) {
                        const uint32_t t = t0 + lane;
                        int k = 0;
#pragma unroll
                        for (int st = 16; st >= 1; st >>= 1) {
                            const uint32_t v = __shfl_sync(FULL, excl, (k + st) & 31);
                            if (k + st < 32 && v <= t) k += st;
                        }
                        const uint32_t ob = __shfl_sync(FULL, cand, k), oe = __shfl_sync(FULL, excl, k);
                        if (t >= tot) continue;
                        const uint32_t x = (uint32_t)(g0 + k) * 32 + select_bit(ob, t - oe);
                        if (WORK) ++w_tests;
                        bool hit = false;
                        uint32_t s0 = __ldg(a.ptr + x), s1 = __ldg(a.ptr + x + 1), j = s0;
                        for (; j < s1 && !hit; ++j) hit = vis_test_ca(P.vis[d], __ldg(a.col + j));
                        if (WORK) w_probes += j - s0;
                        if (!hit && a.dptr) {
                            s0 = __ldg(a.dptr + x);
                            s1 = __ldg(a.dptr + x + 1);
                            for (j = s0; j < s1 && !hit; ++j) hit = vis_test_ca(P.vis[d], __ldg(a.dcol + j));
                            if (WORK) w_probes += j - s0;
                        }
                        if (hit) {
                            atomicOr(&P.vis[d][x >> 5], 1u << (x & 31));
                            atomicOr(&P.nb[d][cb][x >> 5], 1u << (x & 31));
                            ++marks;
                        }
                    }
                }
            }
            ++bu;
        } else if (!td) {
#if DBL_BU_ILP
            // two vertices x both directions per iteration: the four
            // dependent chains (bitmap word -> row pointers -> first
            // neighbour -> its bitmap bit) run interleaved, so a sweep pays
            // about half the serial round trips; most vertices stop at the
            // first neighbour, the rest continue with the serial scan
            for (uint64_t x0 = tid; x0 < P.n; x0 += 2 * nth) {
                uint32_t xv[2], w[2][2], s0[2][2], s1[2][2], c0[2][2];
                bool need[2][2];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint64_t x = x0 + i * nth;
                    xv[i] = (uint32_t)x;
#pragma unroll
                    for (int d = 0; d < 2; ++d)
                        w[i][d] = x < P.n ? *(volatile uint32_t *)&P.vis[d][x >> 5] : ~0u;
                }
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int d = 0; d < 2; ++d) {
                        need[i][d] = !((w[i][d] >> (xv[i] & 31)) & 1u);
                        s0[i][d] = s1[i][d] = 0;
                        if (need[i][d]) {
                            s0[i][d] = __ldg(P.adj[d].ptr + xv[i]);
                            s1[i][d] = __ldg(P.adj[d].ptr + xv[i] + 1);
                        }
                    }
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int d = 0; d < 2; ++d) {
                        c0[i][d] = (need[i][d] && s1[i][d] > s0[i][d]) ? __ldg(P.adj[d].col + s0[i][d]) : 0xffffffffu;
                        DBL_DCHECK(c0[i][d] == 0xffffffffu || c0[i][d] < P.n);
                    }
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int d = 0; d < 2; ++d) {
                        if (!need[i][d]) continue;
                        if (WORK) ++w_tests;
                        bool hit = c0[i][d] != 0xffffffffu && vis_test_ca(P.vis[d], c0[i][d]);
                        uint32_t pr = c0[i][d] != 0xffffffffu;
                        if (!hit) {
                            const Adj &a = P.adj[d];
                            uint32_t j = s0[i][d] + 1;
                            for (; j < s1[i][d] && !hit; ++j)
                                hit = vis_test_ca(P.vis[d], __ldg(a.col + j));
                            if (WORK) pr += j > s0[i][d] + 1 ? j - s0[i][d] - 1 : 0;
                            if (!hit && a.dptr) {
                                const uint32_t t0 = __ldg(a.dptr + xv[i]), t1 = __ldg(a.dptr + xv[i] + 1);
                                uint32_t jd = t0;
                                for (; jd < t1 && !hit; ++jd) hit = vis_test_ca(P.vis[d], __ldg(a.dcol + jd));
                                if (WORK) pr += jd - t0;
                            }
                        }
                        if (WORK) w_probes += pr;
                        if (hit) {
                            atomicOr(&P.vis[d][xv[i] >> 5], 1u << (xv[i] & 31));
                            atomicOr(&P.nb[d][cb][xv[i] >> 5], 1u << (xv[i] & 31));
                            ++marks;
                        }
                    }
            }
#else
            for (uint64_t x = tid; x < P.n; x += nth) {
#pragma unroll
                for (int d = 0; d < 2; ++d) {
                    const uint32_t w = *(volatile uint32_t *)&P.vis[d][x >> 5];
                    if ((w >> (x & 31)) & 1u) continue;
                    if (any_marked(P.adj[d], P.vis[d], (uint32_t)x)) {
                        atomicOr(&P.vis[d][x >> 5], 1u << (x & 31));
                        atomicOr(&P.nb[d][cb][x >> 5], 1u << (x & 31));
                        ++marks;
                    }
                }
            }
#endif
            ++bu;
        } else {
            const int pb = (step + 2) % 3;   // the previous step's marks
#pragma unroll
            for (int d = 0; d < 2; ++d) {
                const Adj &a = P.top[d];
                for (uint64_t wi = tid; wi < P.nwords; wi += nth) {
                    uint32_t f = P.nb[d][pb][wi];
                    while (f) {
                        const uint32_t y = (uint32_t)(wi * 32 + __ffs(f) - 1);
                        f &= f - 1;
                        if (WORK) ++w_tdv;
#pragma unroll 1
                        for (int seg = 0; seg < 2; ++seg) {
                            const uint32_t *ptr = seg ? a.dptr : a.ptr;
                            if (!ptr) break;
                            const uint32_t *col = seg ? a.dcol : a.col;
                            const uint32_t s0 = __ldg(ptr + y), s1 = __ldg(ptr + y + 1);
                            if (WORK) w_tde += s1 - s0;
                            for (uint32_t j = s0; j < s1; ++j) {
                                const uint32_t z = __ldg(col + j);
                                DBL_DCHECK(z < P.n);
                                const uint32_t bit = 1u << (z & 31);
                                if (vis_test_ca(P.vis[d], z)) continue;
                                if (!(atomicOr(&P.vis[d][z >> 5], bit) & bit)) {
                                    atomicOr(&P.nb[d][cb][z >> 5], bit);
                                    ++marks;
                                }
                            }
                        }
                    }
                }
            }
        }
        // clear the bitmaps step s + 1 writes (written in s - 2, read in s - 1)
        const int clr = (step + 1) % 3;
        for (uint64_t wi = tid; wi < P.nwords; wi += nth) { P.nb[0][clr][wi] = 0; P.nb[1][clr][wi] = 0; }
        for (int o = 16; o > 0; o >>= 1) marks += __shfl_xor_sync(FULL, marks, o);
        if ((threadIdx.x & 31) == 0 && marks) atomicAdd(&P.changed[cb], marks);
        if (tid == 0) P.changed[(step + 1) % 3] = 0;
        grid.sync();
        const unsigned got = *(volatile unsigned int *)&P.changed[cb];
        if (P.tr && tid == 0 && step < 32) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            P.tr[2 * step] = t;
            P.tr[2 * step + 1] = got | ((unsigned long long)td << 32);
        }
        if (!got) {
            if (tid == 0) { P.changed[4] = step + 1; P.changed[5] = bu; }
            break;
        }
        // switch on the shrinking tail only: a growing frontier (a pivot with
        // few neighbours, uniform random graphs: cfg1) stays bottom-up --
        // top-down levels take one thread per bitmap word and serialise on
        // large frontiers (cfg1: 0.25 -> 1.06 ms when it switched at step 0)
        if (!td && step >= 1 && got < P.td_switch && got < prev_got) td = true;
        prev_got = got;
    }
    if (WORK) {   // one warp-aggregated add per counter per warp
        unsigned long long c[4] = {w_tests, w_probes, w_tdv, w_tde};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            for (int o = 16; o > 0; o >>= 1) c[i] += __shfl_xor_sync(FULL, c[i], o);
            if ((threadIdx.x & 31) == 0 && c[i]) atomicAdd(&P.work[i], c[i]);
        }
    }
    // keep D(h) and the SCC landmarks for query pruning (marks are exact
    // members even when the sweeps were capped)
    if (P.dmask_out)
        for (uint64_t w = tid; w < P.nwords; w += nth) P.dmask_out[w] = P.vis[0][w];
    if (P.scc_out)
        for (uint64_t i = tid; i < P.k; i += nth) {
            const uint32_t x = P.lm[i];
            if (x < P.n && (((P.vis[0][x >> 5] & P.vis[1][x >> 5]) >> (x & 31)) & 1u))
                atomicOr(&P.scc_out[i / 64], 1ull << (i % 64));
        }
    // a capped search without both level-0 bitmaps drops the head start
    // (grid-uniform); the records are still written when they are not yet
    const bool drop = capped && !(P.front[0] && P.front[1]);
    if (drop && !P.write_rec) return;
    // L_in(h) = OR of the in-halves over A(h), L_out(h) = OR of the
    // out-halves over D(h); then every x in D(h) takes L_in(h), every x in
    // A(h) takes L_out(h)
    __shared__ unsigned long long acc[2 * MAX_SHARD_WORDS];
    const uint32_t H = P.H, rw = 2 * H, rs = rec_stride(H);
    const uint64_t wm = capped ? P.cap_wmask : P.wmask;
    for (uint32_t i = threadIdx.x; i < rw; i += blockDim.x) acc[i] = 0;
    __syncthreads();
    // The records hold exactly the seeds (or are about to), so the unions come from the
    // metadata (5 coalesced bytes per vertex instead of the records): source
    // leaves and landmarks in A(h) give L_in(h), sinks and landmarks in D(h)
    // give L_out(h) (seeding as in prep_kernel / landmark_seed_kernel).
    if (!drop) {
        const uint32_t wdl = P.wdl, wbl = H - wdl;
        const int lane = threadIdx.x & 31;
        const uint64_t nr = ((uint64_t)P.n + 31) & ~31ull;   // warp-uniform trips
        for (uint64_t x = tid; x < nr; x += nth) {
            uint32_t qin = 0xffffffffu, qout = 0xffffffffu, bb = 0;
            if (x < P.n) {
                const uint8_t f = P.flags[x];
                if (f) {
                    const uint32_t b = P.bucket[x];
                    bb = b % 64;
                    if ((f & 1) && ((P.vis[1][x >> 5] >> (x & 31)) & 1u)) qin = b / 64;
                    if ((f & 2) && ((P.vis[0][x >> 5] >> (x & 31)) & 1u)) qout = b / 64;
                }
            }
            if (!__any_sync(FULL, qin != 0xffffffffu || qout != 0xffffffffu)) continue;
            bool full = true;
            for (uint32_t q = 0; q < wbl; ++q) {
                const uint64_t vi = qin == q ? 1ull << bb : 0ull, vo = qout == q ? 1ull << bb : 0ull;
                const uint64_t ri = ((uint64_t)__reduce_or_sync(FULL, (uint32_t)(vi >> 32)) << 32) |
                                    __reduce_or_sync(FULL, (uint32_t)vi);
                const uint64_t ro = ((uint64_t)__reduce_or_sync(FULL, (uint32_t)(vo >> 32)) << 32) |
                                    __reduce_or_sync(FULL, (uint32_t)vo);
                if (lane == 0) {
                    // every bucket bit of the word present: this CTA's share
                    // of the union is complete (R-MAT: after a few hundred
                    // leaves of its ~57k vertices at cfg5)
                    const uint64_t fm = (q == wbl - 1 && P.kp % 64) ? (1ull << (P.kp % 64)) - 1 : ~0ull;
                    uint64_t got_in = fm, got_out = fm;
                    if ((wm >> (wdl + q)) & 1u)
                        got_in = (ri ? atomicOr(&acc[wdl + q], (unsigned long long)ri) : acc[wdl + q]) | ri;
                    if ((wm >> (H + wdl + q)) & 1u)
                        got_out = (ro ? atomicOr(&acc[H + wdl + q], (unsigned long long)ro) : acc[H + wdl + q]) | ro;
                    full = full && (got_in & fm) == fm && (got_out & fm) == fm;
                }
            }
            if (__shfl_sync(FULL, full, 0)) break;
        }
        for (uint64_t i = tid; i < P.k; i += nth) {
            const uint32_t x = P.lm[i], w = (uint32_t)(i / 64);
            if (x >= P.n) continue;
            const unsigned long long bit = 1ull << (i % 64);
            if (((P.vis[1][x >> 5] >> (x & 31)) & 1u) && ((wm >> w) & 1u)) atomicOr(&acc[w], bit);
            if (((P.vis[0][x >> 5] >> (x & 31)) & 1u) && ((wm >> (H + w)) & 1u)) atomicOr(&acc[H + w], bit);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < rw; i += blockDim.x)
        if (acc[i]) atomicOr(&P.L[i], acc[i]);
    // large graphs: the unions are complete when the kernel ends, and
    // reach_apply_kernel (launched behind it) writes them into the records;
    // small ones apply here (a launch costs more than their apply)
    if (!P.fused_apply) return;
    grid.sync();
    for (uint32_t i = threadIdx.x; i < rw; i += blockDim.x) acc[i] = *(volatile unsigned long long *)&P.L[i];
    __syncthreads();
    apply_head_start<WORK, 0>(P, tid, nth, acc, drop, capped);
    if (P.write_rec) {   // landmark i seeds bit i of both DL halves (labels.py:291-293)
        grid.sync();
        for (uint64_t i = tid; i < P.k; i += nth) {
            const uint32_t x = P.lm[i];
            if (x >= P.n) continue;
            const unsigned long long bit = 1ull << (i % 64);
            atomicOr(reinterpret_cast<unsigned long long *>(P.rec + (uint64_t)x * rs + i / 64), bit);
            atomicOr(reinterpret_cast<unsigned long long *>(P.rec + (uint64_t)x * rs + H + i / 64), bit);
        }
    }
}

// Apply the head start (after reach_kernel; a plain launch at full occupancy,
// no grid barrier: the records stream out at HBM write rate).
template <bool WORK, int MODE>
__global__ void __launch_bounds__(256) reach_apply_kernel(ReachParams P) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    const bool have = P.lm[0] < P.n;
    if (!have && !P.write_rec) return;
    const bool capped = *(volatile unsigned int *)&P.changed[3] != 0;
    const bool drop = capped && !(P.front[0] && P.front[1]);
    if (drop && !P.write_rec) return;
    __shared__ unsigned long long acc[2 * MAX_SHARD_WORDS];
    const uint32_t H = P.H, rw = 2 * H, rs = rec_stride(H);
    for (uint32_t i = threadIdx.x; i < rw; i += blockDim.x) acc[i] = drop ? 0ull : P.L[i];
    __syncthreads();
    apply_head_start<WORK, MODE>(P, tid, nth, acc, drop, capped);
    if (!P.write_rec) return;
    // landmark i seeds bit i of both DL halves (labels.py:291-293) once every
    // record is written whole: the last CTA to finish ORs them in
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&P.changed[6], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (uint32_t i = threadIdx.x; i < P.k; i += blockDim.x) {
        const uint32_t x = P.lm[i];
        if (x >= P.n) continue;
        const unsigned long long bit = 1ull << (i % 64);
        atomicOr(reinterpret_cast<unsigned long long *>(P.rec + (uint64_t)x * rs + i / 64), bit);
        atomicOr(reinterpret_cast<unsigned long long *>(P.rec + (uint64_t)x * rs + H + i / 64), bit);
    }
}

static bool pivot_on() { return !DBL_NO_PIVOT; }

// Head start from the pivot's reachability (all record words; after prep).
static dbl_status pivot_head_start(dbl_graph *g, dbl_index *idx, uint64_t wmask, uint32_t *front0,
                                   uint32_t *front1, uint64_t cap_wmask, bool write_rec,
                                   const uint32_t *haspred = nullptr) {
    const uint32_t n = g->n, H = idx->wdl + idx->wbl;
    const size_t bmw = ((size_t)n + 31) / 32;
    const size_t bbytes = ((bmw * 4 + 255) / 256) * 256;
    dbl_status s;
    const size_t rbytes = 8 * bbytes + 2 * MAX_SHARD_WORDS * 8 + 64 + 66 * 8 + 16 * 8;
    if ((s = g->reach.ensure(rbytes))) return s;
    uint32_t *vf = g->reach.as<uint32_t>();
    uint32_t *vb = reinterpret_cast<uint32_t *>(g->reach.as<char>() + bbytes);
    unsigned long long *L = reinterpret_cast<unsigned long long *>(g->reach.as<char>() + 8 * bbytes);
    unsigned int *chg = reinterpret_cast<unsigned int *>(L + 2 * MAX_SHARD_WORDS);
    DBL_CUDA(cudaMemsetAsync(g->reach.p, 0, rbytes, g->stream));
    ReachParams R{};
    R.rec = idx->rec.as<uint64_t>();
    R.L = L;
    R.wmask = wmask;
    R.cap_wmask = cap_wmask;
    R.front[0] = front0;
    R.front[1] = front1;
    R.k = idx->cfg.k;
    R.kp = idx->cfg.k_prime;
    R.haspred[0] = haspred;
    R.haspred[1] = haspred ? haspred + bmw : nullptr;
    R.wdl = idx->wdl;
    R.dmask_out = nullptr;
    R.scc_out = nullptr;
    if (wmask == ~0ull) {   // full builds keep the pivot sets for query pruning
        if ((s = idx->dmask.ensure(bmw * 4 + 64)) || (s = idx->sccmask.ensure((size_t)idx->wdl * 8 + 16))) return s;
        DBL_CUDA(cudaMemsetAsync(idx->sccmask.p, 0, (size_t)idx->wdl * 8 + 16, g->stream));
        R.dmask_out = idx->dmask.as<uint32_t>();
        R.scc_out = idx->sccmask.as<unsigned long long>();
        idx->dmask_n = n;
        idx->has_scc = true;
    }
    R.H = H;
    R.adj[0] = graph_rev(g);
    R.adj[1] = graph_fwd(g);
    R.top[0] = graph_fwd(g);
    R.top[1] = graph_rev(g);
    R.vis[0] = vf;
    R.vis[1] = vb;
    for (int d = 0; d < 2; ++d)
        for (int j = 0; j < 3; ++j)
            R.nb[d][j] = reinterpret_cast<uint32_t *>(g->reach.as<char>() + (2 + 3 * d + j) * bbytes);
    R.changed = chg;
    R.lm = idx->landmarks.as<uint32_t>();
    R.flags = idx->leaf_flags.as<uint8_t>();
    R.bucket = idx->bucket.as<uint32_t>();
    R.write_rec = write_rec;
    R.n = n;
    R.nwords = (uint32_t)bmw;
    // bottom-up sweeps cost O(n) each: shallow graphs (R-MAT, d >= 4) finish
    // in ~5; deep sparse ones stop here and hand the partial sets to the
    // label fixpoint's frontier
    R.max_sweeps = 12;
#ifndef DBL_REACH_MAX_STEPS
#define DBL_REACH_MAX_STEPS 64
#endif
    R.max_steps = DBL_REACH_MAX_STEPS;
    R.td_switch = DBL_TD_DIV ? (uint32_t)(n / DBL_TD_DIV) : 0u;
    constexpr bool tr = DBL_TRACE;
    unsigned long long *trb = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(chg) + 64);
    R.tr = tr ? trb : nullptr;
    // the instrumented variant (dbl_graph_instrument) counts the executed
    // work; the product variant carries no counters (they cost registers)
    const bool wk = g->instrument;
    R.work = trb + 66;
    g->reach_work = wk ? R.work : nullptr;
    g->reach_chg = chg;
    const bool big = n >= (1u << 24);
    const void *kern = big ? (wk ? (const void *)reach_kernel<8, true> : (const void *)reach_kernel<8, false>)
                           : (wk ? (const void *)reach_kernel<6, true> : (const void *)reach_kernel<6, false>);
    int bps = 1;
    if ((s = kernel_occupancy(kern, 256, 0, &bps))) return s;
    {   // at least ~2 word groups per warp and direction (cfg2: 4 words, cfg5: 32)
        const uint64_t warps = (uint64_t)g->sm_count * bps * 8;
        uint32_t gsz = 32;
        while (gsz > 1 && (uint64_t)bmw < warps * gsz * 2) gsz >>= 1;
        R.sparse_g = gsz;
    }
    // the records stream out faster from a separate full-occupancy kernel
    // once they are large (cfg5: 1.64 vs ~2.2 ms); a small graph's apply is
    // cheaper than a launch (cfg2: ~14 us either way)
    R.fused_apply = (uint64_t)n * idx->rs * 8 < (256ull << 20);
    void *args[] = {(void *)&R};
    DBL_CUDA(cudaLaunchCooperativeKernel(kern, dim3(g->sm_count * bps), dim3(256), args, 0, g->stream));
    DBL_LAUNCHED();
    if (!R.fused_apply) {
        // one resident wave (grid-stride over the 32-vertex blocks)
        // write mode with a stride dividing 128 words: 32-byte stores (own
        // kernel: the path's extra registers cost the 16-byte path occupancy)
        const bool v32 = write_rec && idx->rs >= 8 && 128 % idx->rs == 0;
        const void *ak = wk ? (v32 ? (const void *)reach_apply_kernel<true, 2> : (const void *)reach_apply_kernel<true, 1>)
                            : (v32 ? (const void *)reach_apply_kernel<false, 2> : (const void *)reach_apply_kernel<false, 1>);
        int abps = 1;
        if ((s = kernel_occupancy(ak, 256, 0, &abps))) return s;
        const uint64_t blocks_needed = ((uint64_t)bmw * 32 + 255) / 256;
        const uint64_t full = (uint64_t)g->sm_count * abps;
        const int ag = (int)(blocks_needed < full ? (blocks_needed ? blocks_needed : 1) : full);
        void *aargs[] = {(void *)&R};
        DBL_CUDA(cudaLaunchKernel(ak, dim3(ag), dim3(256), aargs, 0, g->stream));
        DBL_CHECK_LAUNCH("reach_apply_kernel");
    }
    if (DBL_TRACE) {
        unsigned int hc[6];
        DBL_CUDA(cudaMemcpyAsync(hc, chg, sizeof(hc), cudaMemcpyDeviceToHost, g->stream));
        DBL_CUDA(cudaStreamSynchronize(g->stream));
        std::fprintf(stderr, "[dbl] pivot reach: %u steps, %u bottom-up%s\n", hc[4], hc[5],
                     hc[3] ? " (cap hit: partial sets)" : "");
        unsigned long long ht[66];
        DBL_CUDA(cudaMemcpy(ht, trb, sizeof(ht), cudaMemcpyDeviceToHost));
        unsigned long long prev = ht[64];
        for (uint32_t st = 0; st < hc[4] && st < 32; ++st) {
            std::fprintf(stderr, "[dbl]   step %2u %s marks %9u  %8.1f us\n", st, (ht[2 * st + 1] >> 32) ? "TD" : "BU",
                         (unsigned)ht[2 * st + 1], (ht[2 * st] - prev) / 1000.0);
            prev = ht[2 * st];
        }
    }
    return DBL_OK;
}

// Build (or rebuild) the listed record words (nullptr = all) from seeds.
// A full build seeds through the fused prep pass (select.cu: metadata still
// to be selected, seeds, level-0 frontier of the first word group, device
// landmark top-k), so nothing between the graph and the fixpoint waits on
// the host; a word subset (sharded builds) seeds with seed_records.
dbl_status run_build(dbl_graph *g, dbl_index *idx, const uint32_t *words, uint32_t nwords) {
    if (idx->n == 0) return DBL_OK;
    Group groups[2 * MAX_SHARD_WORDS + 4];
    int ng = 0;
    if (idx->wdl + idx->wbl > (uint32_t)MAX_SHARD_WORDS) { set_error("label width too large"); return DBL_E_CONFIG; }
    plan_groups(idx, words, nwords, groups, ng);
    // pair forward and backward groups of equal width into one launch
    const Group *pairs[2 * MAX_SHARD_WORDS + 4][2];
    int np = 0;
    {
        bool used[2 * MAX_SHARD_WORDS + 4] = {};
        for (int i = 0; i < ng; ++i) {
            if (used[i]) continue;
            used[i] = true;
            pairs[np][0] = pairs[np][1] = nullptr;
            pairs[np][groups[i].dir] = &groups[i];
            for (int j = i + 1; j < ng; ++j) {
                if (!used[j] && groups[j].dir != groups[i].dir && groups[j].nw == groups[i].nw) {
                    used[j] = true;
                    pairs[np][groups[j].dir] = &groups[j];
                    break;
                }
            }
            ++np;
        }
    }
    DBL_CUDA(cudaEventRecord(g->ev[0], g->stream));
    idx->has_scc = false;   // set again by a full build's pivot
    const bool prep = words == nullptr;
    g->last_build = BuildWork{};
    g->reach_work = nullptr;
    dbl_status s;
    if ((s = graph_ensure_traversal(g))) return s;
    // a full build with a pivot lets the pivot pass write the seeded records
    // (one write of the table instead of seed + read-modify-write)
    constexpr bool rec_in_prep = DBL_PREP_RECORDS;
    const bool pivot = idx->cfg.k && pivot_on();
    // (measured: wins on padded k = 256 records, cfg5 9.3 -> 8.4 ms; costs ~4 us
    // on 32-byte records, cfg2, where prep's write is cheap)
    const bool pivot_writes = prep && pivot && !rec_in_prep && idx->rs > 4;
    g->last_build.flags = (prep && !pivot_writes ? 1u : 0u) | (pivot_writes ? 2u : 0u) |
                          (pivot && !pivot_writes ? 4u : 0u) | (prep ? 0u : 16u);
    g->last_build.rs = idx->rs;
    bool haspred_ok = false;
    if (prep) {
        const Group **p0 = pairs[0];
        uint32_t *b0 = p0[0] ? g->stamp[0].as<uint32_t>() : nullptr;
        uint32_t *b1 = p0[1] ? g->stamp[1].as<uint32_t>() : nullptr;
        // has-predecessor bitmaps for the sparse later sweeps: they pay from
        // 2^21 vertices on (2^24: 1.32 -> 1.22 ms per build, cfg5 5.51 ->
        // 5.07 ms); on cfg2 the dense sweep is faster (13.4 vs 15.4 us)
        const bool want_hp = pivot && g->n >= (1u << 21);
        if (want_hp && (s = g->haspred.ensure((((size_t)g->n + 31) / 32) * 8 + 64))) return s;
        if ((s = prep_build_dev(g, idx, b0, b1, p0[0] ? p0[0]->w0 : 0, p0[0] ? p0[0]->w0 + p0[0]->nw : 0,
                                p0[1] ? p0[1]->w0 : 0, p0[1] ? p0[1]->w0 + p0[1]->nw : 0, !pivot_writes,
                                want_hp ? g->haspred.as<uint32_t>() : nullptr, &haspred_ok)))
            return s;
    } else {
        uint64_t wmask = 0;
        for (uint32_t i = 0; i < nwords; ++i) wmask |= 1ull << words[i];
        if ((s = index_seed_records(g, idx, wmask))) return s;
    }
    trace("build: seed", g->stream);
    if (pivot) {
        uint64_t wmask = ~0ull;
        if (!prep) {
            wmask = 0;
            for (uint32_t i = 0; i < nwords; ++i) wmask |= 1ull << words[i];
        }
        // prep wrote the first word group's level-0 bitmaps (all words are
        // covered by the head start then): prune h's SCC from them
        uint32_t *f0 = nullptr, *f1 = nullptr;
        uint64_t cap_wmask = 0;
        if (prep) {
            f0 = pairs[0][0] ? g->stamp[0].as<uint32_t>() : nullptr;
            f1 = pairs[0][1] ? g->stamp[1].as<uint32_t>() : nullptr;
            for (int d = 0; d < 2; ++d)
                if (pairs[0][d])
                    for (uint32_t w = pairs[0][d]->w0; w < pairs[0][d]->w0 + pairs[0][d]->nw; ++w) cap_wmask |= 1ull << w;
        }
        if ((s = pivot_head_start(g, idx, wmask, f0, f1, cap_wmask, pivot_writes,
                                  haspred_ok ? g->haspred.as<uint32_t>() : nullptr)))
            return s;
        // (the capped case needs both bitmaps; with a one-direction first
        // group the kernel drops the head start instead)
        trace("build: pivot head start", g->stream);
    }
    PrepState hp{};
    for (int pi = 0; pi < np; ++pi) {
        const Group *pair[2] = {pairs[pi][0], pairs[pi][1]};
        const bool fresh = !(prep && pi == 0);   // prep wrote pair 0's level-0 bitmaps
        FixParams P{};
        uint32_t nw = 0;
        bool vec = true;
        if ((s = prepare_params(g, idx, pair, P, nw, vec, false, true, fresh))) return s;
        if (fresh && (s = launch_init_frontier(g, idx, pair))) return s;
        trace("build: init frontier", g->stream);
        if ((s = launch_fixpoint<false>(g, P, nw, vec))) return s;
        Ctrl h{};
        if ((s = finish_run(g, &h, prep && pi == 0 ? &hp : nullptr))) return s;
        trace("build: fixpoint", g->stream);
        g->last_build.fix_runs += 1;
        g->last_build.fix_levels += h.levels;
        for (uint32_t l = 0; l < h.levels && l < 32; ++l) {
            g->last_build.fix_items += h.level_items[l] & ((1ull << 60) - 1);
            g->last_build.fix_edges += h.level_edges[l];
        }
        if (prep && pi == 0) {
            if (hp.err) { set_error("bucket override outside [0, k_prime)"); return DBL_E_CONFIG; }
            idx->sel_leaves = false;
            idx->ovr.release();
            if (hp.fallback) {
                // more landmark candidates than the on-chip sort holds (flat
                // score distributions): exact top-k with the radix-sort path,
                // then build again from the fixed metadata
                if ((s = select_landmarks_dev(g, idx->cfg.k, idx->cfg.strategy, idx->landmarks.as<uint32_t>())))
                    return s;
                idx->sel_landmarks = false;
                return run_build(g, idx, words, nwords);
            }
            idx->sel_landmarks = false;
        }
        if (DBL_TRACE) {
#if DBL_TRACE
            {
                unsigned long long cp[5] = {0, 0, 0, 0, 0};
                cudaMemcpyFromSymbol(cp, g_compact_prof, sizeof(cp));
                unsigned long long z[5] = {0, 0, 0, 0, 0};
                cudaMemcpyToSymbol(g_compact_prof, z, sizeof(z));
                const double tot = (double)(cp[0] + cp[1] + cp[2] + cp[3] + cp[4]) + 1;
                std::fprintf(stderr, "[dbl] compaction cycles (all levels): bits+scan %.0f%%, select %.0f%%, row ptrs %.0f%%, reserve %.0f%%, stores %.0f%%  (%.3g warp-cycles)\n",
                             100 * cp[0] / tot, 100 * cp[1] / tot, 100 * cp[2] / tot, 100 * cp[3] / tot, 100 * cp[4] / tot, tot);
            }
#endif
            std::fprintf(stderr, "[dbl] fixpoint levels=%u nw=%u  level-0 compaction per warp: max %.1f us, mean %.1f us, last start %.1f us after level start\n",
                         h.levels, nw, h.dbg[0] / 1e3, h.dbg[1] / 1e3 / (g->sm_count * 8.0 * 4), (h.dbg[3] - h.level_t[0]) / 1e3);
            for (uint32_t l = 0; l < h.levels && l < 31; ++l)
                std::fprintf(stderr, "[dbl]   level %2u items %9llu edges %10llu pull %llu compact %7.1f us  relax %7.1f us\n",
                             l, h.level_items[l] & ((1ull << 60) - 1), h.level_edges[l], h.level_items[l] >> 60,
                             (h.level_t[2 * l + 1] - h.level_t[2 * l]) / 1e3,
                             (h.level_t[2 * l + 2] - h.level_t[2 * l + 1]) / 1e3);
        }
    }
    // ev[1] was recorded (and reached) by the last finish_run
    cudaEventElapsedTime(&g->t_fix, g->ev[0], g->ev[1]);
    return DBL_OK;
}

// Propagate a batch of new edges (sorted forward keys, already added to the
// graph) through all label words.
dbl_status run_insert(dbl_graph *g, dbl_index *idx, const uint64_t *new_keys, uint64_t count,
                      bool count_changes, uint32_t *changed_out, uint32_t *seed_changed,
                      uint32_t *levels, const unsigned long long *extra_dev, unsigned long long *extra_host,
                      const uint64_t *dcount) {
    changed_out[0] = changed_out[1] = 0;
    seed_changed[0] = seed_changed[1] = 0;
    *levels = 0;
    g->last_insert = BuildWork{};
    if (count == 0 || idx->n == 0) return DBL_OK;
    Group groups[2 * MAX_SHARD_WORDS + 4];
    int ng = 0;
    plan_groups(idx, nullptr, 0, groups, ng);
    DBL_CUDA(cudaEventRecord(g->ev[0], g->stream));
    // groups come ordered: dir 0 groups then dir 1 groups with equal widths
    const int half = ng / 2;
    for (int i = 0; i < half; ++i) {
        const Group *pair[2] = {&groups[i], &groups[half + i]};
        FixParams P{};
        uint32_t nw = 0;
        bool vec = true;
        dbl_status s = prepare_params(g, idx, pair, P, nw, vec, count_changes, i == 0);
        if (s) return s;
        trace("insert: params", g->stream);
        if ((s = launch_insert_seed(g, P, nw, vec, count_changes, new_keys, count, dcount))) return s;
        trace("insert: seed launched", g->stream);
        if (count_changes) {
            if ((s = launch_fixpoint<true>(g, P, nw, vec))) return s;
        } else {
            if ((s = launch_fixpoint<false>(g, P, nw, vec))) return s;
        }
        trace("insert: fixpoint launched", g->stream);
        Ctrl h{};
        // the caller's extra device word (batch stats) rides on the last sync
        const bool last = i == half - 1;
        if ((s = finish_run(g, &h, nullptr, last ? extra_dev : nullptr, last ? extra_host : nullptr))) return s;
        trace("insert: fixpoint", g->stream);
        if (DBL_TRACE) {
            std::fprintf(stderr, "[dbl] insert fixpoint levels=%u nw=%u\n", h.levels, nw);
            for (uint32_t l = 0; l < h.levels && l < 31; ++l)
                std::fprintf(stderr, "[dbl]   level %2u items %9llu edges %10llu compact %7.1f us  relax %7.1f us\n",
                             l, h.level_items[l] & ((1ull << 60) - 1), h.level_edges[l],
                             (h.level_t[2 * l + 1] - h.level_t[2 * l]) / 1e3,
                             (h.level_t[2 * l + 2] - h.level_t[2 * l + 1]) / 1e3);
        }
        // the change bitmap persists across groups, so counts stay distinct
        changed_out[0] += (uint32_t)h.changed[0];
        changed_out[1] += (uint32_t)h.changed[1];
        seed_changed[0] |= h.seed_changed[0];
        seed_changed[1] |= h.seed_changed[1];
        if (h.levels > *levels) *levels = h.levels;
        g->last_insert.fix_runs += 1;
        g->last_insert.fix_levels += h.levels;
        for (uint32_t l = 0; l < h.levels && l < 32; ++l) {
            g->last_insert.fix_items += h.level_items[l] & ((1ull << 60) - 1);
            g->last_insert.fix_edges += h.level_edges[l];
        }
    }
    // ev[1] was recorded (and reached) by the last finish_run
    cudaEventElapsedTime(&g->t_fix, g->ev[0], g->ev[1]);
    return DBL_OK;
}

// ------------------------------------------------------------- work model --
// level-synchronous (Jacobi) counts per 64-bit family.

__global__ void wm_extract_kernel(const uint64_t *__restrict__ rec, uint32_t rs, uint32_t w, uint32_t n,
                                  uint64_t *__restrict__ cur, uint8_t *__restrict__ front) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint64_t x = rec[(size_t)v * rs + w];
        cur[v] = x;
        front[v] = x != 0;
    }
}

__global__ void wm_push_kernel(Adj adj, uint32_t n, const uint64_t *__restrict__ cur,
                               const uint8_t *__restrict__ front, uint64_t *__restrict__ nxt,
                               unsigned long long *__restrict__ VE) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long V = 0, E = 0;
    for (uint64_t v = warp; v < n; v += nwarps) {
        if (!front[v]) continue;
        const uint64_t lab = cur[v];
        uint32_t s = adj.ptr[v], e = adj.ptr[v + 1];
        uint32_t ds = 0, de = 0;
        if (adj.dptr) { ds = adj.dptr[v]; de = adj.dptr[v + 1]; }
        if (lane == 0) { V += 1; E += (e - s) + (de - ds); }
        for (uint32_t i = s + lane; i < e; i += 32) atomicOr((unsigned long long *)&nxt[adj.col[i]], lab);
        for (uint32_t i = ds + lane; i < de; i += 32) atomicOr((unsigned long long *)&nxt[adj.dcol[i]], lab);
    }
    if (lane == 0) {
        atomicAdd(&VE[0], V);
        atomicAdd(&VE[1], E);
    }
}

__global__ void wm_diff_kernel(uint32_t n, uint64_t *__restrict__ cur, const uint64_t *__restrict__ nxt,
                               uint8_t *__restrict__ front) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint64_t a = cur[v], b = nxt[v];
        front[v] = a != b;
        cur[v] = b;
    }
}

dbl_status work_model(const dbl_index *idx, dbl_graph *g, uint64_t *V, uint64_t *E, uint32_t *levels) {
    const uint32_t n = idx->n, rw = idx->rw, rs = idx->rs, H = idx->wdl + idx->wbl;
    DevBuf seeds, cur, nxt, front, ve;
    dbl_index tmp;  // seed records only
    dbl_status s;
    auto cleanup = [&]() { seeds.release(); cur.release(); nxt.release(); front.release(); ve.release(); };
    if ((s = seeds.ensure((size_t)n * rs * 8 + 16)) || (s = cur.ensure((size_t)n * 8 + 8)) ||
        (s = nxt.ensure((size_t)n * 8 + 8)) || (s = front.ensure((size_t)n + 8)) || (s = ve.ensure(16))) {
        cleanup();
        return s;
    }
    // seed records into `seeds`
    std::swap(tmp.rec, seeds);
    tmp.n = n; tmp.rw = rw; tmp.rs = rs; tmp.wdl = idx->wdl; tmp.wbl = idx->wbl; tmp.cfg = idx->cfg;
    tmp.landmarks.p = idx->landmarks.p;
    tmp.leaf_flags.p = idx->leaf_flags.p;
    tmp.bucket.p = idx->bucket.p;
    s = index_seed_records(g, &tmp, ~0ull);
    std::swap(tmp.rec, seeds);
    tmp.landmarks.p = tmp.leaf_flags.p = tmp.bucket.p = nullptr;
    if (s) { cleanup(); return s; }
    const int blocks = g->sm_count * 8;
    for (uint32_t w = 0; w < rw; ++w) {
        Adj adj = w < H ? graph_fwd(g) : graph_rev(g);
        wm_extract_kernel<<<blocks, 256, 0, g->stream>>>(seeds.as<uint64_t>(), rs, w, n, cur.as<uint64_t>(),
                                                         front.as<uint8_t>());
        DBL_LAUNCHED();
        uint64_t Vt = 0, Et = 0;
        uint32_t L = 0;
        for (;;) {
            unsigned long long h[2];
            DBL_CUDA(cudaMemsetAsync(ve.p, 0, 16, g->stream));
            DBL_CUDA(cudaMemcpyAsync(nxt.p, cur.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, g->stream));
            wm_push_kernel<<<blocks, 256, 0, g->stream>>>(adj, n, cur.as<uint64_t>(), front.as<uint8_t>(),
                                                          nxt.as<uint64_t>(), ve.as<unsigned long long>());
            DBL_LAUNCHED();
            DBL_CUDA(cudaMemcpyAsync(h, ve.p, 16, cudaMemcpyDeviceToHost, g->stream));
            DBL_CUDA(cudaStreamSynchronize(g->stream));
            if (h[0] == 0) break;
            Vt += h[0];
            Et += h[1];
            ++L;
            wm_diff_kernel<<<blocks, 256, 0, g->stream>>>(n, cur.as<uint64_t>(), nxt.as<uint64_t>(),
                                                          front.as<uint8_t>());
            DBL_LAUNCHED();
        }
        V[w] = Vt;
        E[w] = Et;
        levels[w] = L;
    }
    cleanup();
    return DBL_OK;
}

}  // namespace dbl
