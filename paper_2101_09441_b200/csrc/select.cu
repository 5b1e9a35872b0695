// select.cu -- K1 landmark ranking and K2 leaf selection / leaf hashing.
//
// select_landmarks (reference labels.py:140-147) orders vertices by
// (-score, id) and keeps the top k; the score is LandmarkStrategy.score
// (labels.py:39-46) of (in-degree, out-degree), computed here as u64, which
// is exact for n < 2^32.  A stable descending radix sort over the scores of
// vertices listed in id order reproduces the (-score, id) tie-break exactly.
//
// select_leaves (labels.py:150-181) + leaf_hash (labels.py:119-137): one
// thread per vertex, splitmix64 mix mod k' in u64 wrap-around arithmetic.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace dbl {

__host__ __device__ __forceinline__ uint32_t leaf_hash_u64(uint64_t v, uint32_t k_prime, uint64_t seed) {
    uint64_t x = v * 0x9E3779B97F4A7C15ull + seed * 0xD1B54A32D192ED03ull;
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return (uint32_t)(x % (uint64_t)k_prime);
}

// The same hash with the final 64-bit modulo as a multiply-high by
// magic = floor((2^64 - 1) / k') and one correction (the quotient estimate
// is at most one short), exact for every x and k' >= 1: the general 64-bit
// division is the most expensive part of the build's prep pass.
__device__ __forceinline__ uint32_t leaf_hash_magic(uint64_t v, uint32_t k_prime, uint64_t magic, uint64_t seed_mix) {
    uint64_t x = v * 0x9E3779B97F4A7C15ull + seed_mix;
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    uint64_t r = x - __umul64hi(x, magic) * k_prime;
    if (r >= k_prime) r -= k_prime;
    return (uint32_t)r;
}

__global__ void leaf_hash_kernel(const uint64_t *__restrict__ ids, uint64_t count, uint32_t k_prime,
                                 uint64_t seed, uint32_t *__restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = leaf_hash_u64(ids[i], k_prime, seed);
}

dbl_status leaf_hash_dev(const uint64_t *ids, uint64_t count, uint32_t k_prime, uint64_t seed,
                         uint32_t *out, cudaStream_t s) {
    if (!count) return DBL_OK;
    int blocks = (int)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
    leaf_hash_kernel<<<blocks, 256, 0, s>>>(ids, count, k_prime, seed, out);
    DBL_CHECK_LAUNCH("leaf_hash_kernel");
    return DBL_OK;
}

__device__ __forceinline__ uint64_t strategy_score(int strategy, uint64_t in, uint64_t out) {
    switch (strategy) {
    case DBL_STRAT_MAX: return in > out ? in : out;
    case DBL_STRAT_MIN: return in < out ? in : out;
    case DBL_STRAT_SUM: return in + out;
    default: return in * out;
    }
}

// bin 0: score 0; bin i (1..64): floor(log2(score)) + 1
__device__ __forceinline__ int score_bin(uint64_t s) { return s ? 64 - __clzll((long long)s) : 0; }

// score[v] for every vertex + a 65-bin log2 histogram of the scores
__global__ void score_hist_kernel(const uint32_t *__restrict__ fptr, const uint32_t *__restrict__ rptr,
                                  const uint32_t *__restrict__ dfptr, const uint32_t *__restrict__ drptr,
                                  uint32_t n, int strategy, uint64_t *__restrict__ score,
                                  uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[65];
    for (int i = threadIdx.x; i < 65; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        uint64_t out = fptr[v + 1] - fptr[v], in = rptr[v + 1] - rptr[v];
        if (dfptr) { out += dfptr[v + 1] - dfptr[v]; in += drptr[v + 1] - drptr[v]; }
        const uint64_t sc = strategy_score(strategy, in, out);
        score[v] = sc;
        atomicAdd(&h[score_bin(sc)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 65; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

struct BinAtLeast {
    const uint64_t *score;
    int bin;
    __device__ bool operator()(uint32_t v) const { return score_bin(score[v]) >= bin; }
};

__global__ void gather_scores_kernel(const uint64_t *__restrict__ score, const uint32_t *__restrict__ ids,
                                     uint32_t c, uint64_t *__restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x)
        out[i] = score[ids[i]];
}

// Top-k by (-score, id): a log2 histogram finds the lowest score bin that
// still holds the k-th best vertex; only vertices in that bin or above can be
// landmarks.  They are compacted in id order and stable-sorted by score
// descending, which reproduces sorted(key=(-score, id)) (labels.py:145-146).
dbl_status select_landmarks_dev(dbl_graph *g, uint32_t k, int strategy, uint32_t *dev_out) {
    uint32_t n = g->n;
    if (k > n) { set_error("k exceeds vertex count"); return DBL_E_CONFIG; }
    if (k == 0) return DBL_OK;
    dbl_status s;
    const size_t nb = (size_t)n * 8;
    if ((s = g->scratch_a.ensure(nb * 2 + 65 * 4 + 64)) || (s = g->scratch_b.ensure((size_t)n * 8 + 64))) return s;
    uint64_t *sc = g->scratch_a.as<uint64_t>(), *sc_sorted_a = sc + n;
    uint32_t *hist = reinterpret_cast<uint32_t *>(sc + 2 * (size_t)n);
    uint32_t *ids = g->scratch_b.as<uint32_t>(), *ids2 = ids + n;
    Adj f = graph_fwd(g), r = graph_rev(g);
    DBL_CUDA(cudaMemsetAsync(hist, 0, 65 * 4, g->stream));
    int blocks = (int)((n + 255) / 256 < (uint32_t)g->sm_count * 8 ? (n + 255) / 256 : g->sm_count * 8);
    score_hist_kernel<<<blocks, 256, 0, g->stream>>>(f.ptr, r.ptr, f.dptr, r.dptr, n, strategy, sc, hist);
    DBL_CHECK_LAUNCH("score_hist_kernel");
    uint32_t hh[65];
    DBL_CUDA(cudaMemcpyAsync(hh, hist, sizeof(hh), cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    int bin = 64;
    uint64_t acc = 0;
    for (; bin >= 0; --bin) {
        acc += hh[bin];
        if (acc >= k) break;
    }
    if (bin < 0) bin = 0;
    // candidates in id order
    if ((s = g->scratch_c.ensure(16))) return s;
    int *d_nsel = g->scratch_c.as<int>();
    cub::CountingInputIterator<uint32_t> it(0);
    size_t tmp = 0;
    BinAtLeast pred{sc, bin};
    DBL_CUDA(cub::DeviceSelect::If(nullptr, tmp, it, ids, d_nsel, (int64_t)n, pred, g->stream));
    if ((s = g->cub_tmp.ensure(tmp))) return s;
    DBL_CUDA(cub::DeviceSelect::If(g->cub_tmp.p, tmp, it, ids, d_nsel, (int64_t)n, pred, g->stream));
    DBL_LAUNCHED();
    int c = 0;
    DBL_CUDA(cudaMemcpyAsync(&c, d_nsel, 4, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    uint64_t *csc = sc_sorted_a, *csc2 = csc + c;   // candidate scores (c <= n)
    if ((size_t)c * 2 > (size_t)n) {                 // large candidate set: reuse score buffer layout
        if ((s = g->scratch_d.ensure((size_t)c * 16 + 16))) return s;
        csc = g->scratch_d.as<uint64_t>();
        csc2 = csc + c;
    }
    gather_scores_kernel<<<(c + 255) / 256 < 4096 ? (c + 255) / 256 : 4096, 256, 0, g->stream>>>(sc, ids, c, csc);
    DBL_CHECK_LAUNCH("gather_scores_kernel");
    cub::DoubleBuffer<uint64_t> dk(csc, csc2);
    cub::DoubleBuffer<uint32_t> dv(ids, ids2);
    tmp = 0;
    DBL_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, dk, dv, (int64_t)c, 0, 64, g->stream));
    if ((s = g->cub_tmp.ensure(tmp))) return s;
    DBL_CUDA(cub::DeviceRadixSort::SortPairsDescending(g->cub_tmp.p, tmp, dk, dv, (int64_t)c, 0, 64, g->stream));
    DBL_LAUNCHED();
    DBL_CUDA(cudaMemcpyAsync(dev_out, dv.Current(), (size_t)k * 4, cudaMemcpyDeviceToDevice, g->stream));
    return DBL_OK;
}

__global__ void leaves_kernel(const uint32_t *__restrict__ fptr, const uint32_t *__restrict__ rptr,
                              const uint32_t *__restrict__ dfptr, const uint32_t *__restrict__ drptr,
                              uint32_t n, uint64_t threshold, uint32_t k_prime, uint64_t seed,
                              const uint32_t *__restrict__ ovr, uint8_t *__restrict__ flags,
                              uint32_t *__restrict__ bucket, unsigned long long *err) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        uint64_t out = fptr[v + 1] - fptr[v], in = rptr[v + 1] - rptr[v];
        if (dfptr) { out += dfptr[v + 1] - dfptr[v]; in += drptr[v + 1] - drptr[v]; }
        uint8_t f = 0;
        if (in == 0) f |= 1;
        if (out == 0) f |= 2;
        if (threshold > 0 && in * out <= threshold) f |= 3;
        uint32_t b = 0;
        if (f) {
            uint32_t o = ovr ? ovr[v] : 0xffffffffu;
            if (o != 0xffffffffu) {
                if (o >= k_prime) atomicOr(err, 1ull);
                b = o;
            } else {
                b = leaf_hash_u64(v, k_prime, seed);
            }
        }
        flags[v] = f;
        bucket[v] = b;
    }
}

dbl_status select_leaves_dev(dbl_graph *g, uint64_t threshold, uint32_t k_prime, uint64_t seed,
                             const uint32_t *dev_ovr, uint8_t *dev_flags, uint32_t *dev_bucket) {
    if (k_prime < 1) { set_error("k_prime must be >= 1"); return DBL_E_CONFIG; }
    uint32_t n = g->n;
    if (n == 0) return DBL_OK;
    dbl_status s = g->scratch_c.ensure(16);
    if (s) return s;
    unsigned long long *err = g->scratch_c.as<unsigned long long>();
    DBL_CUDA(cudaMemsetAsync(err, 0, 8, g->stream));
    Adj f = graph_fwd(g), r = graph_rev(g);
    int blocks = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    leaves_kernel<<<blocks, 256, 0, g->stream>>>(f.ptr, r.ptr, f.dptr, r.dptr, n, threshold, k_prime,
                                                 seed, dev_ovr, dev_flags, dev_bucket, err);
    DBL_CHECK_LAUNCH("leaves_kernel");
    unsigned long long herr = 0;
    DBL_CUDA(cudaMemcpyAsync(&herr, err, 8, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    if (herr) { set_error("bucket override outside [0, k_prime)"); return DBL_E_CONFIG; }
    return DBL_OK;
}

// ------------------------------------------------- fused build prep (K1-K3) --
//
// One pass over the vertices replaces score_hist + leaves + seed_records +
// leaf_frontier (four launches and two host round trips): degrees ->
// landmark score and its log2 histogram, leaf flags and buckets (labels.py:
// 150-181), the seeded record (labels.py:291-305 seeding) and the level-0
// frontier bitmaps.  The landmark top-k then runs without the host: a
// candidate pass keeps every vertex whose score bin can still hold a
// landmark, and one CTA sorts the candidates by (-score, id) in shared memory
// (labels.py:145-146) and ORs the landmark bits into the records/bitmaps.

struct PrepArgs {
    Adj f, r;
    uint32_t n;
    int strategy;
    int do_lm, do_leaves;
    uint64_t threshold;
    uint32_t k_prime;
    uint64_t seed;
    uint64_t kp_magic, seed_mix;   // leaf_hash_magic constants
    uint8_t *bins;                 // score bin per vertex (landmark candidates)
    uint32_t *hp0, *hp1;           // has-predecessor bitmaps (in-degree > 0, out-degree > 0), or nullptr
    const uint32_t *ovr;
    uint8_t *flags;
    uint32_t *bucket;
    uint64_t *rec;
    uint32_t wdl, wbl;
    uint32_t *bits0, *bits1;
    uint32_t a0, e0, a1, e1;
    PrepState *st;
};

// LM: landmark scores + histogram; LV: leaf selection (else the flags and
// buckets are read); DL: the graph has delta adjacency.  Warp-uniform
// switches as template parameters: the pass is issue-bound, not HBM-bound.
template <bool LM, bool LV, bool DL>
__global__ void __launch_bounds__(256) prep_kernel(const PrepArgs A) {
    __shared__ uint32_t h[65];
    if (LM) {
        for (int i = threadIdx.x; i < 65; i += blockDim.x) h[i] = 0;
        __syncthreads();
    }
    const uint32_t H = A.wdl + A.wbl, rw = 2 * H, rs = rec_stride(H);
    const uint64_t nr = ((uint64_t)A.n + 31) & ~31ull;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    // A warp takes 32 consecutive vertices per step; each lane loads row
    // pointer i and takes i + 1 from its neighbour (lane 31 loads it), and
    // the next step's pointers load while this step is processed.
    constexpr bool degs = LM || LV;
    const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t nf0 = 0, nf1 = 0, nr0 = 0, nr1 = 0;
    auto fetch = [&](uint64_t i) {
        nf0 = i <= A.n ? __ldg(A.f.ptr + i) : 0u;
        nr0 = i <= A.n ? __ldg(A.r.ptr + i) : 0u;
        if (lane == 31 && i < A.n) {
            nf1 = __ldg(A.f.ptr + i + 1);
            nr1 = __ldg(A.r.ptr + i + 1);
        }
    };
    if (degs && i0 < nr) fetch(i0);
    for (uint64_t i = i0; i < nr; i += stride) {
        const bool valid = i < A.n;
        const uint32_t v = (uint32_t)i;
        uint8_t f = 0;
        uint32_t b = 0;
        uint32_t out = 1, in = 1;   // (unknown without degs: every leaf joins the frontier)
        if (degs) {
            uint32_t cf1 = __shfl_down_sync(FULL, nf0, 1), cr1 = __shfl_down_sync(FULL, nr0, 1);
            if (lane == 31) { cf1 = nf1; cr1 = nr1; }
            out = cf1 - nf0;
            in = cr1 - nr0;
            if (i + stride < nr) fetch(i + stride);
            if (DL && valid) { out += A.f.dptr[v + 1] - A.f.dptr[v]; in += A.r.dptr[v + 1] - A.r.dptr[v]; }
            if (LM) {
                // bin 0 (a degree-0 end: ~70% of R-MAT vertices) counted by
                // one ballot; the other lanes aggregate per bin
                const int bin = valid ? score_bin(strategy_score(A.strategy, in, out)) : 0;
                if (valid) A.bins[v] = (uint8_t)bin;
                const unsigned z = __ballot_sync(FULL, valid && bin == 0);
                const unsigned nz = __ballot_sync(FULL, valid && bin != 0);
                if (lane == 0 && z) atomicAdd(&h[0], (uint32_t)__popc(z));
                if (valid && bin != 0) {
                    const unsigned peers = __match_any_sync(nz, bin);
                    if (lane == __ffs(peers) - 1) atomicAdd(&h[bin], (uint32_t)__popc(peers));
                }
            }
            if (LV && valid) {
                f = (in == 0 ? 1 : 0) | (out == 0 ? 2 : 0);
                if (A.threshold > 0 && (uint64_t)in * out <= A.threshold) f = 3;
                if (f) {
                    const uint32_t o = A.ovr ? A.ovr[v] : 0xffffffffu;
                    if (o != 0xffffffffu) {
                        if (o >= A.k_prime) atomicOr(&A.st->err, 1ull);
                        b = o;
                    } else {
                        b = leaf_hash_magic(v, A.k_prime, A.kp_magic, A.seed_mix);
                    }
                }
                A.flags[v] = f;
                A.bucket[v] = b;
            }
        }
        if (!LV && valid) {
            f = A.flags[v];
            b = A.bucket[v];
        }
        // seeds: bl_in bit for source leaves, bl_out bit for sinks, dl words 0
        const uint32_t bw = A.wdl + b / 64;
        const uint32_t win = (f & 1) ? bw : 0xffffffffu;
        const uint32_t wout = (f & 2) ? H + bw : 0xffffffffu;
        const uint64_t bit = 1ull << (b % 64);
        // a leaf joins the level-0 frontier of a direction only if it has
        // edges to push along (R-MAT: 57% of the vertices are source leaves,
        // 10% have out-edges; the rest would only cost compaction work)
        const bool p0 = (f & 1) && out > 0 && bw >= A.a0 && bw < A.e0;
        const bool p1 = (f & 2) && in > 0 && H + bw >= A.a1 && H + bw < A.e1;
        // the warp's 32 records (pad words included) as one contiguous block
        // (skipped when the pivot pass writes the records: A.rec == nullptr):
        // each store instruction covers 512 bytes, whole sectors and lines
        // (per-record 16-byte stores at the record stride are partial-sector
        // writes, which cost L2 read-fills)
        if (A.rec && rs <= 4) {
            // one-sector records: the thread's own two 16-byte stores complete
            // its sector (no partial-sector fills)
            if (valid) {
                uint64_t *r = A.rec + i * rs;
                for (uint32_t w = 0; w < rw; w += 2) {
                    ulonglong2 val;
                    val.x = (w == win || w == wout) ? bit : 0ull;
                    val.y = (w + 1 == win || w + 1 == wout) ? bit : 0ull;
                    *reinterpret_cast<ulonglong2 *>(r + w) = val;
                }
            }
        } else if (A.rec) {
            const uint64_t v0 = i - lane;
            uint64_t *blk = A.rec + v0 * rs;
            for (uint32_t t = 0; t < rs * 32; t += 64) {
                const uint32_t wi = t + 2 * lane, r = wi / rs, w = wi % rs;
                const uint32_t swin = __shfl_sync(FULL, win, r), swout = __shfl_sync(FULL, wout, r);
                const uint64_t sbit = ((uint64_t)__shfl_sync(FULL, (uint32_t)(bit >> 32), r) << 32) |
                                      __shfl_sync(FULL, (uint32_t)bit, r);
                if (v0 + r < A.n) {
                    ulonglong2 val;
                    val.x = (w == swin || w == swout) ? sbit : 0ull;
                    val.y = (w + 1 == swin || w + 1 == swout) ? sbit : 0ull;
                    *reinterpret_cast<ulonglong2 *>(blk + wi) = val;
                }
            }
        }
        const unsigned b0 = __ballot_sync(FULL, p0), b1 = __ballot_sync(FULL, p1);
        unsigned h0 = 0, h1 = 0;
        if (degs) {
            h0 = __ballot_sync(FULL, valid && in > 0);
            h1 = __ballot_sync(FULL, valid && out > 0);
        }
        if (lane == 0) {
            if (A.bits0) A.bits0[i >> 5] = b0;
            if (A.bits1) A.bits1[i >> 5] = b1;
            if (degs && A.hp0) {
                A.hp0[i >> 5] = h0;
                A.hp1[i >> 5] = h1;
            }
        }
    }
    if (LM) {
        __syncthreads();
        for (int i = threadIdx.x; i < 65; i += blockDim.x)
            if (h[i]) atomicAdd(&A.st->hist[i], h[i]);
    }
}

// Candidates of the top-k: every vertex whose score bin is at or above the
// lowest bin that still holds the k-th best score (bins from the histogram;
// each CTA derives the threshold itself).  Unordered; at most
// PREP_CAND_CAP are stored, the count is exact.
__global__ void __launch_bounds__(256) topk_candidates_kernel(const Adj f, const Adj r, int strategy,
                                                              const uint8_t *__restrict__ bins, uint32_t n,
                                                              uint32_t k, PrepState *st,
                                                              uint64_t *__restrict__ cs, uint32_t *__restrict__ ci) {
    __shared__ int tbin;
    if (threadIdx.x == 0) {
        uint64_t acc = 0;
        int bin = 64;
        for (; bin >= 0; --bin) {
            acc += st->hist[bin];
            if (acc >= k) break;
        }
        tbin = bin < 0 ? 0 : bin;
    }
    __syncthreads();
    const uint32_t t = (uint32_t)tbin;
    const int lane = threadIdx.x & 31;
    // 16 bins per thread per step (one 16-byte load); a warp reserves the
    // slots of all its candidates with one atomicAdd, and a candidate's score
    // is recomputed from its degrees (there are at most a few thousand)
    const uint64_t n16 = ((uint64_t)n + 15) / 16, n16r = (n16 + 31) & ~31ull;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n16r; j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t take = 0;
        if (j < n16) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(bins) + j);
            const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (((wv[e >> 2] >> (8 * (e & 3))) & 0xffu) >= t && j * 16 + e < n) take |= 1u << e;
        }
        const uint32_t cnt = __popc(take);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t tot = __shfl_sync(FULL, incl, 31);
        if (!tot) continue;
        uint32_t base = 0;
        if (lane == 31) base = atomicAdd(&st->n_above, tot);
        uint32_t pos = __shfl_sync(FULL, base, 31) + incl - cnt;
        for (; take; take &= take - 1, ++pos) {
            if (pos >= PREP_CAND_CAP) break;
            const uint32_t v = (uint32_t)(j * 16 + __ffs(take) - 1);
            uint64_t out = f.ptr[v + 1] - f.ptr[v], in = r.ptr[v + 1] - r.ptr[v];
            if (f.dptr) { out += f.dptr[v + 1] - f.dptr[v]; in += r.dptr[v + 1] - r.dptr[v]; }
            cs[pos] = strategy_score(strategy, in, out);
            ci[pos] = v;
        }
    }
}

__device__ __forceinline__ bool lm_better(uint64_t sa, uint32_t ia, uint64_t sb, uint32_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// One CTA: bitonic sort of the candidates by (-score, id) in shared memory,
// the first k become the landmarks (position i owns bit i, labels.py:54-74);
// their DL bits go into the seeded records and the level-0 bitmaps.
__global__ void __launch_bounds__(1024) topk_final_kernel(const uint64_t *__restrict__ cs, const uint32_t *__restrict__ ci,
                                                         uint32_t k, PrepState *st, uint32_t *__restrict__ lm,
                                                         uint64_t *__restrict__ rec, uint32_t rs, uint32_t H,
                                                         uint32_t *bits0, uint32_t *bits1, uint32_t a0, uint32_t e0,
                                                         uint32_t a1, uint32_t e1) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t *ss = reinterpret_cast<uint64_t *>(sm);
    uint32_t *si = reinterpret_cast<uint32_t *>(ss + PREP_CAND_CAP);
    const uint32_t c = st->n_above;
    if (c > PREP_CAND_CAP || k > c) {
        if (threadIdx.x == 0) st->fallback = 1;
        return;
    }
    uint32_t p = 1;
    while (p < c) p <<= 1;
    // only the warps the candidate count needs take part (named barrier over
    // nt threads): a 256-candidate sort pays 8-warp barriers, not 32-warp ones
    const uint32_t nt = p < 32 ? 32u : (p < blockDim.x ? p : blockDim.x);
    if (threadIdx.x >= nt) return;
    for (uint32_t i = threadIdx.x; i < p; i += nt) {
        ss[i] = i < c ? cs[i] : 0ull;
        si[i] = i < c ? ci[i] : 0xffffffffu;   // padding sorts after every vertex
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    for (uint32_t kk = 2; kk <= p; kk <<= 1) {
        for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < p; i += nt) {
                const uint32_t x = i ^ j;
                if (x > i) {
                    const bool up = (i & kk) == 0;
                    const bool xb = lm_better(ss[x], si[x], ss[i], si[i]);
                    if (up == xb) {
                        const uint64_t ts = ss[i]; ss[i] = ss[x]; ss[x] = ts;
                        const uint32_t ti = si[i]; si[i] = si[x]; si[x] = ti;
                    }
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
        }
    }
    for (uint32_t i = threadIdx.x; i < k; i += nt) {
        const uint32_t v = si[i], w = i / 64;
        const uint64_t bit = 1ull << (i % 64);
        lm[i] = v;
        if (rec) {
            uint64_t *r = rec + (size_t)v * rs;
            r[w] |= bit;          // dl_in: the landmark reaches itself
            r[H + w] |= bit;      // dl_out
        }
        if (bits0 && w >= a0 && w < e0) atomicOr(&bits0[v >> 5], 1u << (v & 31));
        if (bits1 && H + w >= a1 && H + w < e1) atomicOr(&bits1[v >> 5], 1u << (v & 31));
    }
}

// landmark bits of given (pinned or previously selected) landmarks
__global__ void landmark_seed_kernel(const uint32_t *__restrict__ lm, uint32_t k, uint64_t *__restrict__ rec,
                                     uint32_t rs, uint32_t H, uint32_t *bits0, uint32_t *bits1, uint32_t a0,
                                     uint32_t e0, uint32_t a1, uint32_t e1) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        const uint32_t v = lm[i], w = i / 64;
        const uint64_t bit = 1ull << (i % 64);
        if (rec) {
            atomicOr(reinterpret_cast<unsigned long long *>(rec + (size_t)v * rs + w), bit);
            atomicOr(reinterpret_cast<unsigned long long *>(rec + (size_t)v * rs + H + w), bit);
        }
        if (bits0 && w >= a0 && w < e0) atomicOr(&bits0[v >> 5], 1u << (v & 31));
        if (bits1 && H + w >= a1 && H + w < e1) atomicOr(&bits1[v >> 5], 1u << (v & 31));
    }
}

dbl_status prep_build_dev(dbl_graph *g, dbl_index *idx, uint32_t *bits0, uint32_t *bits1, uint32_t a0,
                          uint32_t e0, uint32_t a1, uint32_t e1, bool write_rec, uint32_t *haspred,
                          bool *haspred_written) {
    const uint32_t n = g->n, k = idx->cfg.k;
    const bool do_lm = idx->sel_landmarks && k > 0;
    if (k > n) { set_error("k exceeds vertex count"); return DBL_E_CONFIG; }
    if (idx->sel_leaves && idx->cfg.k_prime < 1) { set_error("k_prime must be >= 1"); return DBL_E_CONFIG; }
    dbl_status s;
    const size_t cand_bytes = (size_t)PREP_CAND_CAP * 12;
    // the bins need n bytes; the buffer keeps the n x 8 bytes of the former
    // score array: the pivot sweeps behind this pass measured 26 vs 33 us at
    // cfg2 with the smaller allocation (a buffer-placement effect on the
    // later reach buffer, not explained; tools/ab_build.sh)
    if (do_lm && (s = g->scratch_a.ensure((size_t)n * 8 + 64))) return s;
    if ((s = g->prep.ensure(sizeof(PrepState) + 16 + cand_bytes))) return s;
    PrepState *st = g->prep.as<PrepState>();
    uint64_t *cs = reinterpret_cast<uint64_t *>(g->prep.as<char>() + ((sizeof(PrepState) + 15) & ~15ull));
    uint32_t *ci = reinterpret_cast<uint32_t *>(cs + PREP_CAND_CAP);
    DBL_CUDA(cudaMemsetAsync(st, 0, sizeof(PrepState), g->stream));
    PrepArgs A{};
    A.f = graph_fwd(g);
    A.r = graph_rev(g);
    A.n = n;
    A.strategy = idx->cfg.strategy;
    A.do_lm = do_lm;
    A.do_leaves = idx->sel_leaves;
    A.threshold = idx->cfg.leaf_threshold;
    A.k_prime = idx->cfg.k_prime;
    A.seed = idx->cfg.hash_seed;
    A.kp_magic = A.k_prime ? ~0ull / A.k_prime : 0ull;
    A.seed_mix = A.seed * 0xD1B54A32D192ED03ull;
    A.bins = do_lm ? g->scratch_a.as<uint8_t>() : nullptr;
    const bool degs = do_lm || idx->sel_leaves;
    A.hp0 = degs ? haspred : nullptr;
    A.hp1 = degs && haspred ? haspred + (n + 31) / 32 : nullptr;
    if (haspred_written) *haspred_written = A.hp0 != nullptr;
    A.ovr = idx->ovr.p ? idx->ovr.as<uint32_t>() : nullptr;
    A.flags = idx->leaf_flags.as<uint8_t>();
    A.bucket = idx->bucket.as<uint32_t>();
    A.rec = write_rec ? idx->rec.as<uint64_t>() : nullptr;
    A.wdl = idx->wdl;
    A.wbl = idx->wbl;
    A.bits0 = bits0;
    A.bits1 = bits1;
    A.a0 = a0; A.e0 = e0; A.a1 = a1; A.e1 = e1;
    A.st = st;
    int blocks = (int)(((uint64_t)n + 255) / 256);
    if (blocks > g->sm_count * 8) blocks = g->sm_count * 8;
    if (blocks < 1) blocks = 1;
    {
        const int sel = (A.do_lm ? 4 : 0) | (A.do_leaves ? 2 : 0) | (A.f.dptr ? 1 : 0);
        void (*kerns[8])(const PrepArgs) = {prep_kernel<false, false, false>, prep_kernel<false, false, true>,
                                            prep_kernel<false, true, false>,  prep_kernel<false, true, true>,
                                            prep_kernel<true, false, false>,  prep_kernel<true, false, true>,
                                            prep_kernel<true, true, false>,   prep_kernel<true, true, true>};
        kerns[sel]<<<blocks, 256, 0, g->stream>>>(A);
        DBL_CHECK_LAUNCH("prep_kernel");
    }
    const uint32_t H = idx->wdl + idx->wbl;
    if (do_lm) {
        topk_candidates_kernel<<<blocks, 256, 0, g->stream>>>(A.f, A.r, A.strategy, A.bins, n, k, st, cs, ci);
        DBL_CHECK_LAUNCH("topk_candidates_kernel");
        const int fsmem = (int)cand_bytes;
        int fbps = 1;
        dbl_status fs = kernel_occupancy((const void *)topk_final_kernel, 1024, (size_t)fsmem, &fbps);
        if (fs) return fs;
        topk_final_kernel<<<1, 1024, fsmem, g->stream>>>(cs, ci, k, st, idx->landmarks.as<uint32_t>(), A.rec, idx->rs,
                                                         H, bits0, bits1, a0, e0, a1, e1);
        DBL_CHECK_LAUNCH("topk_final_kernel");
    } else if (k) {
        landmark_seed_kernel<<<(k + 255) / 256, 256, 0, g->stream>>>(idx->landmarks.as<uint32_t>(), k, A.rec, idx->rs,
                                                                    H, bits0, bits1, a0, e0, a1, e1);
        DBL_CHECK_LAUNCH("landmark_seed_kernel");
    }
    return DBL_OK;
}

dbl_status prep_fetch(dbl_graph *g, PrepState *host) {
    DBL_CUDA(cudaMemcpyAsync(host, g->prep.p, sizeof(PrepState), cudaMemcpyDeviceToHost, g->stream));
    return DBL_OK;
}

}  // namespace dbl

using namespace dbl;

extern "C" dbl_status dbl_leaf_hash(const uint64_t *ids, uint64_t count, uint32_t k_prime,
                                    uint64_t seed, uint32_t *out, int device) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (k_prime < 1) { set_error("k_prime must be >= 1"); return DBL_E_CONFIG; }
    if (!count) return DBL_OK;
    if (!ids || !out) { set_error("null argument"); return DBL_E_ARG; }
    DBL_CUDA(cudaSetDevice(device));
    set_stream(nullptr);
    DevBuf b;
    dbl_status s = b.ensure(count * 12);
    if (s) return s;
    uint64_t *di = b.as<uint64_t>();
    uint32_t *dout = reinterpret_cast<uint32_t *>(di + count);
    DBL_CUDA(cudaMemcpy(di, ids, count * 8, cudaMemcpyHostToDevice));
    s = leaf_hash_dev(di, count, k_prime, seed, dout, 0);
    if (!s) {
        cudaError_t e = cudaMemcpy(out, dout, count * 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) s = cuda_fail(e, "leaf_hash D2H");
    }
    b.release();
    return s;
}

extern "C" dbl_status dbl_select_landmarks(const dbl_graph *g, uint32_t k, int32_t strategy,
                                           uint32_t *out_ids) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!g || (k && !out_ids)) { set_error("null argument"); return DBL_E_ARG; }
    if (k > g->n) { set_error("k exceeds vertex count"); return DBL_E_CONFIG; }
    if (!k) return DBL_OK;
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    dbl_graph *gm = const_cast<dbl_graph *>(g);
    DevBuf b;
    dbl_status s = b.ensure((size_t)k * 4);
    if (s) return s;
    s = select_landmarks_dev(gm, k, strategy, b.as<uint32_t>());
    if (!s) {
        cudaMemcpyAsync(out_ids, b.p, (size_t)k * 4, cudaMemcpyDeviceToHost, g->stream);
        cudaError_t e = cudaStreamSynchronize(g->stream);
        if (e != cudaSuccess) s = cuda_fail(e, "select_landmarks");
    }
    b.release();
    return s;
}

__global__ void scatter_ovr_kernel(const uint32_t *__restrict__ ids, const uint32_t *__restrict__ b,
                                   uint32_t cnt, uint32_t n, uint32_t *__restrict__ ovr) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        if (ids[i] >= n) continue;  // labels.py:167-171 only consults leaves
        ovr[ids[i]] = b[i];
    }
}

namespace dbl {
// Device override table (n entries, 0xffffffff = none) from host pairs.
dbl_status make_override(dbl_graph *g, const uint32_t *ids, const uint32_t *buckets, uint32_t cnt,
                         DevBuf &ovr) {
    uint32_t n = g->n;
    dbl_status s = ovr.ensure((size_t)n * 4 + (size_t)cnt * 8 + 16);
    if (s) return s;
    uint32_t *o = ovr.as<uint32_t>();
    uint32_t *di = o + n, *db = di + cnt;
    DBL_CUDA(cudaMemsetAsync(o, 0xff, (size_t)n * 4, g->stream));
    if (cnt) {
        // host arrays are copied before this returns (pageable H2D copies
        // are staged synchronously), so the caller may free them
        DBL_CUDA(cudaMemcpyAsync(di, ids, (size_t)cnt * 4, cudaMemcpyHostToDevice, g->stream));
        DBL_CUDA(cudaMemcpyAsync(db, buckets, (size_t)cnt * 4, cudaMemcpyHostToDevice, g->stream));
        scatter_ovr_kernel<<<(cnt + 255) / 256, 256, 0, g->stream>>>(di, db, cnt, n, o);
        DBL_CHECK_LAUNCH("scatter_ovr_kernel");
    }
    return DBL_OK;
}
}  // namespace dbl

extern "C" dbl_status dbl_select_leaves(const dbl_graph *g, uint64_t threshold, uint32_t k_prime,
                                        uint64_t hash_seed, const uint32_t *ovr_ids,
                                        const uint32_t *ovr_buckets, uint32_t n_ovr,
                                        uint8_t *out_flags, uint32_t *out_bucket) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!g || (g->n && (!out_flags || !out_bucket)) || (n_ovr && (!ovr_ids || !ovr_buckets))) {
        set_error("null argument");
        return DBL_E_ARG;
    }
    if (k_prime < 1) { set_error("k_prime must be >= 1"); return DBL_E_CONFIG; }
    uint32_t n = g->n;
    if (!n) return DBL_OK;
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    dbl_graph *gm = const_cast<dbl_graph *>(g);
    DevBuf ovr, outb;
    dbl_status s = DBL_OK;
    const uint32_t *dovr = nullptr;
    if (ovr_ids && n_ovr) {
        s = make_override(gm, ovr_ids, ovr_buckets, n_ovr, ovr);
        dovr = ovr.as<uint32_t>();
    }
    if (!s) s = outb.ensure((size_t)n * 5 + 16);
    if (!s) {
        uint32_t *db = outb.as<uint32_t>();
        uint8_t *df = reinterpret_cast<uint8_t *>(db + n);
        s = select_leaves_dev(gm, threshold, k_prime, hash_seed, dovr, df, db);
        if (!s) {
            cudaMemcpyAsync(out_flags, df, n, cudaMemcpyDeviceToHost, g->stream);
            cudaMemcpyAsync(out_bucket, db, (size_t)n * 4, cudaMemcpyDeviceToHost, g->stream);
            cudaError_t e = cudaStreamSynchronize(g->stream);
            if (e != cudaSuccess) s = cuda_fail(e, "select_leaves D2H");
        }
    }
    ovr.release();
    outb.release();
    return s;
}

// ------------------------------------------------------- R-MAT generator --
// Counter-based R-MAT edge generator for the large synthetic configs: edge i
// at level l draws splitmix64(seed, i, l) (no RNG state), so any slice of the
// edge list can be regenerated independently and the result is deterministic.

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void rmat_kernel(uint32_t scale, uint64_t m, uint64_t seed, uint32_t ta, uint32_t tab, uint32_t tabc,
                            uint32_t *__restrict__ src, uint32_t *__restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0, d = 0;
        const uint64_t base = splitmix64(seed ^ (i * 0xD1B54A32D192ED03ull));
        for (uint32_t l = 0; l < scale; l += 2) {
            const uint64_t r = splitmix64(base + l);
            // two 32-bit uniforms per draw
            for (int h = 0; h < 2 && l + h < scale; ++h) {
                const uint32_t u = (uint32_t)(r >> (32 * h));
                const uint32_t sb = u >= tab;                              // quadrants c, d
                const uint32_t db = (u >= ta && u < tab) || u >= tabc;      // quadrants b, d
                s |= sb << (l + h);
                d |= db << (l + h);
            }
        }
        src[i] = s;
        dst[i] = d;
    }
}

extern "C" dbl_status dbl_rmat_generate(uint32_t scale, uint64_t m, uint64_t seed, double a, double b, double c,
                                        uint32_t *dev_src, uint32_t *dev_dst, int device) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (scale < 1 || scale > 31 || (m && (!dev_src || !dev_dst))) { set_error("bad R-MAT arguments"); return DBL_E_ARG; }
    if (!m) return DBL_OK;
    DBL_CUDA(cudaSetDevice(device));
    auto th = [](double p) { double x = p * 4294967296.0; return (uint32_t)(x >= 4294967295.0 ? 4294967295.0 : x); };
    rmat_kernel<<<148 * 16, 256>>>(scale, m, seed, th(a), th(a + b), th(a + b + c), dev_src, dev_dst);
    DBL_CHECK_LAUNCH("rmat_kernel");
    DBL_CUDA(cudaDeviceSynchronize());
    return DBL_OK;
}
