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

template <int NW, bool VEC>
__device__ __forceinline__ void load_words(const uint64_t *p, uint64_t (&w)[NW]) {
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

// OR the source words into y's words; true iff this thread set a new bit.
template <int NW, bool VEC>
__device__ __forceinline__ bool relax(const DirParams &D, uint32_t y, const uint64_t (&s)[NW]) {
    uint64_t *p = D.lab + (size_t)y * D.stride;
    uint64_t c[NW];
    load_words<NW, VEC>(p, c);
    bool ch = false;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const uint64_t need = s[k] & ~c[k];
        if (need) {
            const uint64_t old = atomicOr(reinterpret_cast<unsigned long long *>(p + k),
                                          (unsigned long long)need);
            ch |= (need & ~old) != 0;
        }
    }
    return ch;
}

template <bool COUNT>
__device__ __forceinline__ void push_changed(const DirParams &D, const Queue &QN, bool ch, uint32_t y,
                                             uint32_t epoch, unsigned long long *cnt_ptr, Ctrl *ctrl,
                                             uint32_t &nchanged) {
    if (!__any_sync(FULL, ch)) return;
    if (COUNT && ch) {
        const uint32_t bit = 1u << (y & 31);
        const uint32_t old = atomicOr(&D.changed_bits[y >> 5], bit);
        if (!(old & bit)) ++nchanged;
    }
    const bool p = ch && (atomicExch(&D.stamp[y], epoch) != epoch);
    warp_enqueue(D, QN, p, y, cnt_ptr, ctrl);
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

__device__ __forceinline__ void red_or(uint64_t *p, uint64_t v) {
    asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Enqueue up to U vertices per lane (ys[r] where ps[r]) with one scan and one
// 64-bit atomicAdd per warp.
template <int U>
__device__ __forceinline__ void warp_enqueue_multi(const DirParams &D, const Queue &QN, const bool (&ps)[U],
                                                   const uint32_t (&ys)[U], unsigned long long *cnt_ptr,
                                                   Ctrl *ctrl) {
    const int lane = threadIdx.x & 31;
    uint32_t b0[U], b1[U], d0[U], d1[U];
    uint32_t ni = 0, ne = 0;
#pragma unroll
    for (int r = 0; r < U; ++r) {
        b0[r] = b1[r] = d0[r] = d1[r] = 0;
        if (ps[r]) {
            b0[r] = __ldg(D.adj.ptr + ys[r]);
            b1[r] = __ldg(D.adj.ptr + ys[r] + 1);
            if (D.adj.dptr) {
                d0[r] = __ldg(D.adj.dptr + ys[r]);
                d1[r] = __ldg(D.adj.dptr + ys[r] + 1);
            }
        }
        ni += (b1[r] > b0[r]) + (d1[r] > d0[r]);
        ne += (b1[r] - b0[r]) + (d1[r] - d0[r]);
    }
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
#pragma unroll
    for (int r = 0; r < U; ++r) {
        if (b1[r] > b0[r]) {
            QN.x[pos] = ys[r]; QN.start[pos] = b0[r]; QN.len[pos] = b1[r] - b0[r]; QN.eoff[pos] = eo;
            ++pos;
            eo += b1[r] - b0[r];
        }
        if (d1[r] > d0[r]) {
            QN.x[pos] = ys[r]; QN.start[pos] = d0[r]; QN.len[pos] = (d1[r] - d0[r]) | DELTA_BIT;
            QN.eoff[pos] = eo;
            ++pos;
            eo += d1[r] - d0[r];
        }
    }
}

// One warp relaxes the edges [e0, e1) of a level's edge space, U rounds of
// 32 consecutive edges at a time: each lane finds its item in a 32-item
// window by a 5-step shuffle search (the window slides forward as edges are
// consumed), then the U column loads, the U destination-label loads and the
// fire-and-forget atomic ORs of the U rounds are issued back to back so their
// latencies overlap.  A destination whose (L2-coherent) read lacked bits is
// pushed: if another thread supplied the bits first the vertex is merely
// re-expanded once with nothing new, which keeps the fixpoint exact.
template <int NW, bool VEC, bool COUNT>
__device__ __forceinline__ void expand_range(const DirParams &D, const Queue &Q, const Queue &QN,
                                             uint32_t nitems, uint32_t e0, uint32_t e1, uint32_t epoch,
                                             unsigned long long *next_cnt, Ctrl *ctrl, uint32_t &nchanged) {
    constexpr int U = NW <= 2 ? 4 : (NW <= 4 ? 2 : 1);
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
            load_words<NW, VEC>(D.lab + (size_t)x * D.stride, w);
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
            }
        }
        uint64_t cur[U][NW];
#pragma unroll
        for (int r = 0; r < U; ++r)
            if (ok[r]) load_words<NW, VEC>(D.lab + (size_t)ys[r] * D.stride, cur[r]);
        bool ps[U];
        bool any = false;
#pragma unroll
        for (int r = 0; r < U; ++r) {
            bool ch = false;
            if (ok[r]) {
                uint64_t *p = D.lab + (size_t)ys[r] * D.stride;
#pragma unroll
                for (int j = 0; j < NW; ++j) {
                    const uint64_t need = src[r][j] & ~cur[r][j];
                    if (need) { red_or(p + j, need); ch = true; }
                }
            }
            ps[r] = ch;
            any |= ch;
        }
        if (!__any_sync(FULL, any)) continue;
#pragma unroll
        for (int r = 0; r < U; ++r) {
            if (COUNT && ps[r]) {
                const uint32_t bit = 1u << (ys[r] & 31);
                const uint32_t old = atomicOr(&D.changed_bits[ys[r] >> 5], bit);
                if (!(old & bit)) ++nchanged;
            }
            if (ps[r]) ps[r] = ld_cg32(D.stamp + ys[r]) != epoch && atomicExch(&D.stamp[ys[r]], epoch) != epoch;
        }
        warp_enqueue_multi<U>(D, QN, ps, ys, next_cnt, ctrl);
    }
}

template <int NW, bool VEC, bool COUNT>
__global__ void __launch_bounds__(FIX_THREADS) fixpoint_kernel(FixParams P) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    Ctrl *ctrl = P.ctrl;
    uint32_t nchanged[2] = {0, 0};
    for (uint32_t L = 0; L < P.max_levels; ++L) {
        const int c3 = L % 3, n3 = (L + 1) % 3, r3 = (L + 2) % 3;
        const unsigned long long q0 = *(volatile unsigned long long *)&ctrl->cnt[c3][0];
        const unsigned long long q1 = *(volatile unsigned long long *)&ctrl->cnt[c3][1];
        if ((q0 | q1) == 0) {
            if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->levels = L;
            break;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctrl->cnt[r3][0] = 0;
            ctrl->cnt[r3][1] = 0;
        }
        const uint32_t n0 = (uint32_t)(q0 >> 32), E0 = (uint32_t)q0;
        const uint32_t n1 = (uint32_t)(q1 >> 32), E1 = (uint32_t)q1;
        const uint64_t total = (uint64_t)E0 + E1;
        // equal edge ranges per warp (multiple of 32)
        uint64_t per = (total + nwarps - 1) / nwarps;
        per = (per + 31) & ~31ull;
        const uint64_t a = (uint64_t)warp * per, b = (a + per < total) ? a + per : total;
        const int par = L & 1;
        const uint32_t epoch = P.epoch0 + L + 1;
        if (a < b) {
            if (a < E0) {
                const DirParams &D = P.d[0];
                expand_range<NW, VEC, COUNT>(D, D.q[par], D.q[par ^ 1], n0, (uint32_t)a,
                                             (uint32_t)(b < E0 ? b : (uint64_t)E0), epoch, &ctrl->cnt[n3][0], ctrl,
                                             nchanged[0]);
            }
            if (b > E0) {
                const DirParams &D = P.d[1];
                const uint32_t s = a > E0 ? (uint32_t)(a - E0) : 0u;
                expand_range<NW, VEC, COUNT>(D, D.q[par], D.q[par ^ 1], n1, s, (uint32_t)(b - E0), epoch,
                                             &ctrl->cnt[n3][1], ctrl, nchanged[1]);
            }
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

// rec := seeds.  bl_in bit bucket[v] for source leaves, bl_out for sinks;
// dl words zero (landmark bits are added by landmark_bits_kernel).
__global__ void seed_records_kernel(uint64_t *__restrict__ rec, uint32_t n, uint32_t wdl, uint32_t wbl,
                                    const uint8_t *__restrict__ flags, const uint32_t *__restrict__ bucket,
                                    uint64_t wmask) {
    const uint32_t rw = 2 * (wdl + wbl), H = wdl + wbl;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)n * rw;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)(i / rw), w = (uint32_t)(i % rw);
        if (!((wmask >> w) & 1)) continue;
        uint64_t val = 0;
        const uint32_t h = w < H ? 0 : 1, ww = w - h * H;
        if (ww >= wdl) {
            const uint8_t f = flags[v];
            const uint32_t b = bucket[v];
            if ((f >> h) & 1) {
                if (b / 64 == ww - wdl) val = 1ull << (b % 64);
            }
        }
        rec[i] = val;
    }
}

__global__ void landmark_bits_kernel(uint64_t *__restrict__ rec, uint32_t rw, uint32_t H,
                                     const uint32_t *__restrict__ lm, uint32_t k, uint64_t wmask) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        const uint64_t v = lm[i];
        if ((wmask >> (i / 64)) & 1)
            atomicOr(reinterpret_cast<unsigned long long *>(rec + v * rw + i / 64), 1ull << (i % 64));
        if ((wmask >> (H + i / 64)) & 1)
            atomicOr(reinterpret_cast<unsigned long long *>(rec + v * rw + H + i / 64), 1ull << (i % 64));
    }
}

// Level-0 frontier: every vertex with a nonzero seed in the group's words.
template <int NW>
__global__ void init_frontier_kernel(FixParams P, uint32_t n, uint32_t active_mask) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t nr = ((uint64_t)n + 31) & ~31ull;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nr; i += stride) {
        const bool valid = i < n;
        const uint32_t v = valid ? (uint32_t)i : 0;
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            if (!((active_mask >> d) & 1)) continue;
            const DirParams &D = P.d[d];
            bool p = false;
            if (valid) {
                const uint64_t *w = D.lab + (size_t)v * D.stride;
                uint64_t acc = 0;
#pragma unroll
                for (int k = 0; k < NW; ++k) acc |= w[k];
                p = acc != 0;
                if (p) D.stamp[v] = P.epoch0;
            }
            warp_enqueue(D, D.q[0], p, v, &P.ctrl->cnt[0][d], P.ctrl);
        }
    }
}

// Insertion seeds (updates.py:129-134 for a whole batch): for each new edge
// u->v, in-words(v) |= in-words(u) and out-words(u) |= out-words(v).
template <int NW, bool VEC, bool COUNT>
__global__ void insert_seed_kernel(FixParams P, const uint64_t *__restrict__ keys, uint64_t count) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t cr = (count + 31) & ~31ull;
    uint32_t nchanged[2] = {0, 0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cr; i += stride) {
        const bool valid = i < count;
        const uint64_t key = valid ? keys[i] : 0;
        const uint32_t u = (uint32_t)(key >> 32), v = (uint32_t)key;
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            const DirParams &D = P.d[d];
            const uint32_t src = d == 0 ? u : v, dst = d == 0 ? v : u;
            bool ch = false;
            if (valid) {
                uint64_t s[NW];
                load_words<NW, VEC>(D.lab + (size_t)src * D.stride, s);
                ch = relax<NW, VEC>(D, dst, s);
                if (ch) atomicOr(&P.ctrl->seed_changed[d], 1u);
            }
            push_changed<COUNT>(D, D.q[0], ch, dst, P.epoch0, &P.ctrl->cnt[0][d], P.ctrl, nchanged[d]);
        }
    }
    if (COUNT) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            uint32_t x = nchanged[d];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
            if (lane == 0 && x) atomicAdd(&P.ctrl->changed[d], (unsigned long long)x);
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
    static int blocks_per_sm = -1;
    if (blocks_per_sm < 0) {
        DBL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, FIX_THREADS, 0));
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    int grid = blocks_per_sm * g->sm_count;
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

static dbl_status launch_init_frontier(dbl_graph *g, FixParams &P, uint32_t nw, uint32_t mask) {
    int blocks = (int)(((uint64_t)g->n + 255) / 256);
    if (blocks > g->sm_count * 8) blocks = g->sm_count * 8;
    if (blocks < 1) blocks = 1;
#define DBL_INIT_CASE(N) case N: init_frontier_kernel<N><<<blocks, 256, 0, g->stream>>>(P, g->n, mask); break;
    switch (nw) {
        DBL_INIT_CASE(1) DBL_INIT_CASE(2) DBL_INIT_CASE(3) DBL_INIT_CASE(4)
        DBL_INIT_CASE(5) DBL_INIT_CASE(6) DBL_INIT_CASE(7) DBL_INIT_CASE(8)
    default: set_error("bad word-group width"); return DBL_E_CONFIG;
    }
#undef DBL_INIT_CASE
    DBL_CHECK_LAUNCH("init_frontier_kernel");
    return DBL_OK;
}

static dbl_status launch_insert_seed(dbl_graph *g, FixParams &P, uint32_t nw, bool vec, bool count,
                                     const uint64_t *keys, uint64_t nk) {
    int blocks = (int)((nk + 255) / 256);
    if (blocks > g->sm_count * 8) blocks = g->sm_count * 8;
    if (blocks < 1) blocks = 1;
#define DBL_SEED_CASE(N)                                                                      \
    case N:                                                                                   \
        if (count) {                                                                          \
            if (vec) insert_seed_kernel<N, (N % 2 == 0), true><<<blocks, 256, 0, g->stream>>>(P, keys, nk); \
            else insert_seed_kernel<N, false, true><<<blocks, 256, 0, g->stream>>>(P, keys, nk); \
        } else {                                                                              \
            if (vec) insert_seed_kernel<N, (N % 2 == 0), false><<<blocks, 256, 0, g->stream>>>(P, keys, nk); \
            else insert_seed_kernel<N, false, false><<<blocks, 256, 0, g->stream>>>(P, keys, nk); \
        }                                                                                     \
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
                                 uint32_t &nw, bool &vec, bool count, bool reset_counts = true) {
    dbl_status s = graph_ensure_traversal(g);
    if (s) return s;
    // stamps: reset when the epoch could wrap during this run
    const uint64_t need = (uint64_t)g->n + 8;
    if ((uint64_t)g->epoch + need >= 0xfffffff0ull) {
        DBL_CUDA(cudaMemsetAsync(g->stamp[0].p, 0, g->stamp[0].bytes, g->stream));
        DBL_CUDA(cudaMemsetAsync(g->stamp[1].p, 0, g->stamp[1].bytes, g->stream));
        g->epoch = 1;
    }
    nw = 0;
    vec = true;
    for (int d = 0; d < 2; ++d) {
        DirParams &D = P.d[d];
        D.adj = d == 0 ? graph_fwd(g) : graph_rev(g);
        D.stride = idx->rw;
        D.stamp = g->stamp[d].as<uint32_t>();
        D.cap = g->qcap;
        for (int p = 0; p < 2; ++p) {
            uint32_t *b = g->qbuf[d][p].as<uint32_t>();
            D.q[p].x = b;
            D.q[p].start = b + g->qcap;
            D.q[p].len = b + 2ull * g->qcap;
            D.q[p].eoff = b + 3ull * g->qcap;
        }
        D.changed_bits = count ? g->changed_bits.as<uint32_t>() + d * (((size_t)g->n + 31) / 32) : nullptr;
        if (gr[d]) {
            D.lab = idx->rec.as<uint64_t>() + gr[d]->w0;
            nw = gr[d]->nw;
            if ((gr[d]->w0 % 2) || (idx->rw % 2)) vec = false;
        } else {
            D.lab = idx->rec.as<uint64_t>();
        }
    }
    P.ctrl = g->ctrl.as<Ctrl>();
    P.epoch0 = g->epoch;
    P.max_levels = g->n + 4;
    DBL_CUDA(cudaMemsetAsync(P.ctrl, 0, sizeof(Ctrl), g->stream));
    if (count && reset_counts)
        DBL_CUDA(cudaMemsetAsync(g->changed_bits.p, 0, (((size_t)g->n + 31) / 32) * 2 * 4, g->stream));
    return DBL_OK;
}

static dbl_status finish_run(dbl_graph *g, Ctrl *hctrl) {
    DBL_CUDA(cudaMemcpyAsync(hctrl, g->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    g->epoch += hctrl->levels + 2;
    if (hctrl->overflow) { set_error("frontier queue overflow"); return DBL_E_CUDA; }
    return DBL_OK;
}

dbl_status index_seed_records(dbl_graph *g, dbl_index *idx, uint64_t wmask) {
    const uint64_t total = (uint64_t)idx->n * idx->rw;
    if (!total) return DBL_OK;
    int blocks = (int)((total + 255) / 256 < (uint64_t)g->sm_count * 16 ? (total + 255) / 256 : g->sm_count * 16);
    seed_records_kernel<<<blocks, 256, 0, g->stream>>>(idx->rec.as<uint64_t>(), idx->n, idx->wdl, idx->wbl,
                                                       idx->leaf_flags.as<uint8_t>(), idx->bucket.as<uint32_t>(),
                                                       wmask);
    DBL_CHECK_LAUNCH("seed_records_kernel");
    if (idx->cfg.k) {
        landmark_bits_kernel<<<(idx->cfg.k + 255) / 256, 256, 0, g->stream>>>(
            idx->rec.as<uint64_t>(), idx->rw, idx->wdl + idx->wbl, idx->landmarks.as<uint32_t>(), idx->cfg.k,
            wmask);
        DBL_CHECK_LAUNCH("landmark_bits_kernel");
    }
    return DBL_OK;
}

// Build (or rebuild) the listed record words (nullptr = all) from seeds.
dbl_status run_build(dbl_graph *g, dbl_index *idx, const uint32_t *words, uint32_t nwords) {
    if (idx->n == 0) return DBL_OK;
    Group groups[2 * MAX_SHARD_WORDS + 4];
    int ng = 0;
    if (idx->wdl + idx->wbl > (uint32_t)MAX_SHARD_WORDS) { set_error("label width too large"); return DBL_E_CONFIG; }
    plan_groups(idx, words, nwords, groups, ng);
    DBL_CUDA(cudaEventRecord(g->ev[0], g->stream));
    uint64_t wmask = ~0ull;
    if (words) {
        wmask = 0;
        for (uint32_t i = 0; i < nwords; ++i) wmask |= 1ull << words[i];
    }
    dbl_status s = index_seed_records(g, idx, wmask);
    if (s) return s;
    trace("build: seed", g->stream);
    // pair forward and backward groups of equal width into one launch
    bool used[2 * MAX_SHARD_WORDS + 4] = {};
    for (int i = 0; i < ng; ++i) {
        if (used[i]) continue;
        used[i] = true;
        const Group *pair[2] = {nullptr, nullptr};
        pair[groups[i].dir] = &groups[i];
        for (int j = i + 1; j < ng; ++j) {
            if (!used[j] && groups[j].dir != groups[i].dir && groups[j].nw == groups[i].nw) {
                used[j] = true;
                pair[groups[j].dir] = &groups[j];
                break;
            }
        }
        FixParams P{};
        uint32_t nw = 0;
        bool vec = true;
        if ((s = prepare_params(g, idx, pair, P, nw, vec, false))) return s;
        const uint32_t mask = (pair[0] ? 1u : 0u) | (pair[1] ? 2u : 0u);
        if ((s = launch_init_frontier(g, P, nw, mask))) return s;
        trace("build: init frontier", g->stream);
        if ((s = launch_fixpoint<false>(g, P, nw, vec))) return s;
        Ctrl h{};
        if ((s = finish_run(g, &h))) return s;
        trace("build: fixpoint", g->stream);
        if (std::getenv("DBL_TRACE")) std::fprintf(stderr, "[dbl] fixpoint levels=%u nw=%u\n", h.levels, nw);
    }
    DBL_CUDA(cudaEventRecord(g->ev[1], g->stream));
    DBL_CUDA(cudaEventSynchronize(g->ev[1]));
    cudaEventElapsedTime(&g->t_fix, g->ev[0], g->ev[1]);
    return DBL_OK;
}

// Propagate a batch of new edges (sorted forward keys, already added to the
// graph) through all label words.
dbl_status run_insert(dbl_graph *g, dbl_index *idx, const uint64_t *new_keys, uint64_t count,
                      bool count_changes, uint32_t *changed_out, uint32_t *seed_changed,
                      uint32_t *levels) {
    changed_out[0] = changed_out[1] = 0;
    seed_changed[0] = seed_changed[1] = 0;
    *levels = 0;
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
        if ((s = launch_insert_seed(g, P, nw, vec, count_changes, new_keys, count))) return s;
        if (count_changes) {
            if ((s = launch_fixpoint<true>(g, P, nw, vec))) return s;
        } else {
            if ((s = launch_fixpoint<false>(g, P, nw, vec))) return s;
        }
        Ctrl h{};
        if ((s = finish_run(g, &h))) return s;
        // the change bitmap persists across groups, so counts stay distinct
        changed_out[0] += (uint32_t)h.changed[0];
        changed_out[1] += (uint32_t)h.changed[1];
        seed_changed[0] |= h.seed_changed[0];
        seed_changed[1] |= h.seed_changed[1];
        if (h.levels > *levels) *levels = h.levels;
    }
    DBL_CUDA(cudaEventRecord(g->ev[1], g->stream));
    DBL_CUDA(cudaEventSynchronize(g->ev[1]));
    cudaEventElapsedTime(&g->t_fix, g->ev[0], g->ev[1]);
    return DBL_OK;
}

// ------------------------------------------------------------- work model --
// level-synchronous (Jacobi) counts per 64-bit family.

__global__ void wm_extract_kernel(const uint64_t *__restrict__ rec, uint32_t rw, uint32_t w, uint32_t n,
                                  uint64_t *__restrict__ cur, uint8_t *__restrict__ front) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint64_t x = rec[(size_t)v * rw + w];
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
    const uint32_t n = idx->n, rw = idx->rw, H = idx->wdl + idx->wbl;
    DevBuf seeds, cur, nxt, front, ve;
    dbl_index tmp;  // seed records only
    dbl_status s;
    auto cleanup = [&]() { seeds.release(); cur.release(); nxt.release(); front.release(); ve.release(); };
    if ((s = seeds.ensure((size_t)n * rw * 8 + 16)) || (s = cur.ensure((size_t)n * 8 + 8)) ||
        (s = nxt.ensure((size_t)n * 8 + 8)) || (s = front.ensure((size_t)n + 8)) || (s = ve.ensure(16))) {
        cleanup();
        return s;
    }
    // seed records into `seeds`
    std::swap(tmp.rec, seeds);
    tmp.n = n; tmp.rw = rw; tmp.wdl = idx->wdl; tmp.wbl = idx->wbl; tmp.cfg = idx->cfg;
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
        wm_extract_kernel<<<blocks, 256, 0, g->stream>>>(seeds.as<uint64_t>(), rw, w, n, cur.as<uint64_t>(),
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
