// query.cu -- K6 label-check kernel and K7 batched pruned-BFS fallback.
//
// Reference: query (queries.py:94-142) and query_batch (queries.py:210-249).
// Rule order per pair (u, v):
//   0 u == v                               REFLEXIVE
//   1 dl_out[u] & dl_in[v]                 DL_POSITIVE
//   2 bl_in[u] & ~bl_in[v] | bl_out[v] & ~bl_out[u]      BL_NEGATIVE
//   3 dl_out[v] & dl_in[u]                 THM1_NEGATIVE
//   4 dl_out[u] & dl_in[u] | dl_out[v] & dl_in[v]        THM2_NEGATIVE
//   5 pruned BFS from u                    BFS_POSITIVE / BFS_NEGATIVE
//
// K6: one query per thread, both AoS records (32 B at k = k' = 64: one sector
// each, two 128-bit loads) gathered through the read-only path; unresolved
// queries are stream-compacted with a warp ballot + one atomicAdd per warp.
//
// K7: 64 unresolved queries share one CTA and one 64-bit word per visited
// vertex (bit i = query i), so an adjacency list read once serves every
// query whose frontier holds that vertex.  Visited/frontier words live in a
// shared-memory hash table; a query leaves the batch as soon as its target
// is found (the target test precedes the visited test, queries.py:131-133).
// Pruning (queries.py:137-140) is evaluated per (vertex, query) against the
// 64 queries' DL/BL words staged in shared memory.  A group whose BFS
// outgrows the table is re-run by the dense variant (direct-mapped global
// arrays), so no query is ever answered on the CPU.
#include "internal.cuh"

namespace dbl {

enum { CNT_PENDING = 0, CNT_ERR = 1, CNT_TICKET = 2, CNT_OVERFLOW = 3, CNT_DTICKET = 4, CNT_WORDS = 8 };
constexpr int GQ = 64;             // queries per BFS group
constexpr int HCAP = 2048;         // shared hash capacity (power of two)
constexpr int HBITS = 11;
constexpr int TCAP = 128;          // target table
constexpr int BFS_THREADS = 256;
constexpr uint32_t EMPTY = 0xffffffffu;
constexpr uint8_t UNRESOLVED = 0xff;

__device__ __forceinline__ void ld_nc128(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}

// ------------------------------------------------------------------ K6 --

template <int WDL, int WBL>
__global__ void __launch_bounds__(256)
label_check_kernel(const uint64_t *__restrict__ rec, uint32_t n, const uint32_t *__restrict__ qu,
                   const uint32_t *__restrict__ qv, uint64_t count, uint32_t flags,
                   uint8_t *__restrict__ codes, uint32_t *__restrict__ visited,
                   uint32_t *__restrict__ pending, uint32_t *__restrict__ counters) {
    constexpr int H = WDL + WBL, RW = 2 * H;
    const bool use_dl = flags & DBL_F_USE_DL, use_bl = flags & DBL_F_USE_BL;
    const bool thm1 = use_dl && (flags & DBL_F_THM1), thm2 = use_dl && (flags & DBL_F_THM2);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t cr = (count + 31) & ~31ull;
    const int lane = threadIdx.x & 31;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cr; i += stride) {
        bool unres = false;
        if (i < count) {
            const uint32_t u = qu[i], v = qv[i];
            uint8_t code = UNRESOLVED;
            if (u >= n || v >= n) {
                atomicOr(&counters[CNT_ERR], 1u);
                code = 0xfe;
            } else if (u == v) {
                code = DBL_REFLEXIVE;
            } else {
                uint64_t a[RW], b[RW];
                const uint64_t *ra = rec + (size_t)u * RW, *rb = rec + (size_t)v * RW;
#pragma unroll
                for (int k = 0; k < RW; k += 2) {
                    ld_nc128(ra + k, a[k], a[k + 1]);
                    ld_nc128(rb + k, b[k], b[k + 1]);
                }
                uint64_t r1 = 0, r3 = 0, r4 = 0, r2 = 0;
#pragma unroll
                for (int k = 0; k < WDL; ++k) {
                    r1 |= a[H + k] & b[k];             // dl_out[u] & dl_in[v]
                    r3 |= b[H + k] & a[k];             // dl_out[v] & dl_in[u]
                    r4 |= (a[H + k] & a[k]) | (b[H + k] & b[k]);
                }
#pragma unroll
                for (int k = 0; k < WBL; ++k)
                    r2 |= (a[WDL + k] & ~b[WDL + k]) | (b[H + WDL + k] & ~a[H + WDL + k]);
                if (use_dl && r1) code = DBL_DL_POSITIVE;
                else if (use_bl && r2) code = DBL_BL_NEGATIVE;
                else if (thm1 && r3) code = DBL_THM1_NEGATIVE;
                else if (thm2 && r4) code = DBL_THM2_NEGATIVE;
            }
            codes[i] = code;
            if (visited) visited[i] = 0;
            unres = code == UNRESOLVED;
        }
        const unsigned m = __ballot_sync(FULL, unres);
        if (m) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&counters[CNT_PENDING], (uint32_t)__popc(m));
            base = __shfl_sync(FULL, base, 0);
            if (unres) pending[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)i;
        }
    }
}

// runtime-width variant (any k, k')
__global__ void __launch_bounds__(256)
label_check_generic(const uint64_t *__restrict__ rec, uint32_t n, uint32_t wdl, uint32_t wbl,
                    const uint32_t *__restrict__ qu, const uint32_t *__restrict__ qv, uint64_t count,
                    uint32_t flags, uint8_t *__restrict__ codes, uint32_t *__restrict__ visited,
                    uint32_t *__restrict__ pending, uint32_t *__restrict__ counters) {
    const uint32_t H = wdl + wbl, RW = 2 * H;
    const bool use_dl = flags & DBL_F_USE_DL, use_bl = flags & DBL_F_USE_BL;
    const bool thm1 = use_dl && (flags & DBL_F_THM1), thm2 = use_dl && (flags & DBL_F_THM2);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t cr = (count + 31) & ~31ull;
    const int lane = threadIdx.x & 31;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cr; i += stride) {
        bool unres = false;
        if (i < count) {
            const uint32_t u = qu[i], v = qv[i];
            uint8_t code = UNRESOLVED;
            if (u >= n || v >= n) {
                atomicOr(&counters[CNT_ERR], 1u);
                code = 0xfe;
            } else if (u == v) {
                code = DBL_REFLEXIVE;
            } else {
                const uint64_t *a = rec + (size_t)u * RW, *b = rec + (size_t)v * RW;
                uint64_t r1 = 0, r2 = 0, r3 = 0, r4 = 0;
                for (uint32_t k = 0; k < wdl; ++k) {
                    const uint64_t ai = __ldg(a + k), ao = __ldg(a + H + k);
                    const uint64_t bi = __ldg(b + k), bo = __ldg(b + H + k);
                    r1 |= ao & bi;
                    r3 |= bo & ai;
                    r4 |= (ao & ai) | (bo & bi);
                }
                for (uint32_t k = 0; k < wbl; ++k)
                    r2 |= (__ldg(a + wdl + k) & ~__ldg(b + wdl + k)) |
                          (__ldg(b + H + wdl + k) & ~__ldg(a + H + wdl + k));
                if (use_dl && r1) code = DBL_DL_POSITIVE;
                else if (use_bl && r2) code = DBL_BL_NEGATIVE;
                else if (thm1 && r3) code = DBL_THM1_NEGATIVE;
                else if (thm2 && r4) code = DBL_THM2_NEGATIVE;
            }
            codes[i] = code;
            if (visited) visited[i] = 0;
            unres = code == UNRESOLVED;
        }
        const unsigned m = __ballot_sync(FULL, unres);
        if (m) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&counters[CNT_PENDING], (uint32_t)__popc(m));
            base = __shfl_sync(FULL, base, 0);
            if (unres) pending[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)i;
        }
    }
}

// ------------------------------------------------------------------ K7 --

constexpr int MAXW = 16;   // max words per label family in the BFS kernel

struct BfsShared {
    uint32_t qidx[GQ];
    uint32_t vcount[GQ];
    uint32_t tkey[TCAP];
    unsigned long long tmask[TCAP];
    unsigned long long done;
    unsigned long long active;
    uint32_t nlist[2];
    uint32_t overflow;
    uint32_t gid;
    uint32_t nq;
};

struct BfsTable {
    uint32_t *key;                 // SMEM only
    unsigned long long *vis;
    unsigned long long *fr[2];
    uint32_t *list[2];
    uint32_t cap;
};

__device__ __forceinline__ uint32_t hash32(uint32_t x) { return x * 0x9E3779B1u; }

template <bool DENSE>
__device__ __forceinline__ int tab_slot(const BfsTable &T, uint32_t x) {
    if (DENSE) return (int)x;
    uint32_t h = hash32(x) >> (32 - HBITS);
#pragma unroll 1
    for (int probe = 0; probe < 64; ++probe) {
        uint32_t k = T.key[h];
        if (k == x) return (int)h;
        if (k == EMPTY) {
            uint32_t old = atomicCAS(&T.key[h], EMPTY, x);
            if (old == EMPTY || old == x) return (int)h;
        }
        h = (h + 1) & (HCAP - 1);
    }
    return -1;
}

template <bool DENSE>
__device__ __forceinline__ uint32_t tab_vertex(const BfsTable &T, int slot) {
    return DENSE ? (uint32_t)slot : T.key[slot];
}

__device__ __forceinline__ unsigned long long tgt_lookup(const BfsShared &S, uint32_t x) {
    uint32_t h = hash32(x) >> 25;  // 7 bits
#pragma unroll 1
    for (int probe = 0; probe < TCAP; ++probe) {
        uint32_t k = S.tkey[h];
        if (k == x) return S.tmask[h];
        if (k == EMPTY) return 0;
        h = (h + 1) & (TCAP - 1);
    }
    return 0;
}

// Runs pruned BFS groups.  SMEM variant: one group per CTA iteration over
// pending[]; DENSE variant: re-runs groups listed in `ovf` with direct-mapped
// global tables (ws: per-CTA slab of n x (3 u64 + 2 u32)).
template <bool DENSE>
__global__ void __launch_bounds__(BFS_THREADS)
bfs_kernel(const uint64_t *__restrict__ rec, uint32_t WDL, uint32_t WBL, uint32_t n, Adj adj,
           const uint32_t *__restrict__ qu, const uint32_t *__restrict__ qv, uint32_t flags,
           const uint32_t *__restrict__ pending, uint32_t *__restrict__ counters,
           uint32_t *__restrict__ ovf, uint8_t *__restrict__ codes, uint32_t *__restrict__ visited,
           char *__restrict__ ws) {
    const uint32_t H = WDL + WBL, rw = 2 * H;
    const uint32_t WD = WDL > 0 ? WDL : 1;
    extern __shared__ __align__(16) unsigned char smem[];
    BfsShared &S = *reinterpret_cast<BfsShared *>(smem);
    unsigned long long *dlo_u = reinterpret_cast<unsigned long long *>(smem + ((sizeof(BfsShared) + 15) & ~15));
    unsigned long long *bli_v = dlo_u + GQ * WD;
    unsigned long long *blo_v = bli_v + GQ * WBL;
    BfsTable T;
    if (DENSE) {
        char *p = ws + (size_t)blockIdx.x * ((size_t)n * 32);
        T.vis = reinterpret_cast<unsigned long long *>(p);
        T.fr[0] = T.vis + n;
        T.fr[1] = T.fr[0] + n;
        T.list[0] = reinterpret_cast<uint32_t *>(T.fr[1] + n);
        T.list[1] = T.list[0] + n;
        T.key = nullptr;
        T.cap = n;
    } else {
        unsigned char *p = reinterpret_cast<unsigned char *>(blo_v + GQ * WBL);
        T.vis = reinterpret_cast<unsigned long long *>(p);
        T.fr[0] = T.vis + HCAP;
        T.fr[1] = T.fr[0] + HCAP;
        T.key = reinterpret_cast<uint32_t *>(T.fr[1] + HCAP);
        T.list[0] = T.key + HCAP;
        T.list[1] = T.list[0] + HCAP;
        T.cap = HCAP;
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const bool use_dl = flags & DBL_F_USE_DL, use_bl = flags & DBL_F_USE_BL;
    const bool prune_dl = use_dl && (flags & DBL_F_PRUNE_DL);
    const bool prune_bl = use_bl && (flags & DBL_F_PRUNE_BL);
    const uint32_t npend = counters[CNT_PENDING];
    const uint32_t ngroups = DENSE ? counters[CNT_OVERFLOW] : (npend + GQ - 1) / GQ;

    for (;;) {
        if (tid == 0) S.gid = atomicAdd(&counters[DENSE ? CNT_DTICKET : CNT_TICKET], 1u);
        __syncthreads();
        const uint32_t gi = S.gid;
        if (gi >= ngroups) break;
        const uint32_t grp = DENSE ? ovf[gi] : gi;
        const uint32_t q0 = grp * GQ;
        const uint32_t nq = min((uint32_t)GQ, npend - q0);
        // clear tables
        const uint32_t clear_n = DENSE ? n : HCAP;
        for (uint32_t s = tid; s < clear_n; s += blockDim.x) {
            T.vis[s] = 0;
            T.fr[0][s] = 0;
            T.fr[1][s] = 0;
            if (!DENSE) T.key[s] = EMPTY;
        }
        for (int s = tid; s < TCAP; s += blockDim.x) { S.tkey[s] = EMPTY; S.tmask[s] = 0; }
        if (tid == 0) {
            S.done = 0;
            S.active = nq == 64 ? ~0ull : ((1ull << nq) - 1);
            S.nlist[0] = 0;
            S.nlist[1] = 0;
            S.overflow = 0;
            S.nq = nq;
        }
        __syncthreads();
        // stage the group's queries
        if (tid < (int)nq) {
            const uint32_t qi = pending[q0 + tid];
            S.qidx[tid] = qi;
            S.vcount[tid] = 0;
            const uint32_t u = qu[qi], v = qv[qi];
            const uint64_t *ru = rec + (size_t)u * rw, *rv = rec + (size_t)v * rw;
            for (uint32_t k = 0; k < WDL; ++k) dlo_u[tid * WD + k] = __ldg(ru + H + k);
            for (uint32_t k = 0; k < WBL; ++k) {
                bli_v[tid * WBL + k] = __ldg(rv + WDL + k);
                blo_v[tid * WBL + k] = __ldg(rv + H + WDL + k);
            }
            // target table: v -> bit tid
            uint32_t h = hash32(v) >> 25;
            for (;;) {
                uint32_t old = atomicCAS(&S.tkey[h], EMPTY, v);
                if (old == EMPTY || old == v) { atomicOr(&S.tmask[h], 1ull << tid); break; }
                h = (h + 1) & (TCAP - 1);
            }
            // source u: visited and level-0 frontier
            const int sl = tab_slot<DENSE>(T, u);
            if (sl < 0) {
                S.overflow = 1;
            } else {
                atomicOr(&T.vis[sl], 1ull << tid);
                if (atomicOr(&T.fr[0][sl], 1ull << tid) == 0) {
                    const uint32_t p = atomicAdd(&S.nlist[0], 1u);
                    T.list[0][p] = (uint32_t)sl;
                }
            }
        }
        __syncthreads();
        int cur = 0;
        for (;;) {
            const uint32_t ncur = S.nlist[cur];
            const unsigned long long act = S.active;
            if (ncur == 0 || (S.done & act) == act || S.overflow) break;
            const int nxt = cur ^ 1;
            for (uint32_t e = warp; e < ncur; e += nwarps) {
                const int slot = (int)T.list[cur][e];
                unsigned long long fw = 0;
                if (lane == 0) {
                    fw = T.fr[cur][slot] & ~*(volatile unsigned long long *)&S.done;
                    T.fr[cur][slot] = 0;
                }
                fw = __shfl_sync(FULL, fw, 0);
                if (fw == 0) continue;
                const uint32_t w = tab_vertex<DENSE>(T, slot);
                if (lane == 0) {
                    unsigned long long m = fw;
                    while (m) {
                        const int b = __ffsll((long long)m) - 1;
                        m &= m - 1;
                        atomicAdd(&S.vcount[b], 1u);
                    }
                }
#pragma unroll 1
                for (int seg = 0; seg < 2; ++seg) {
                    uint32_t s0, s1;
                    const uint32_t *col;
                    if (seg == 0) { s0 = adj.ptr[w]; s1 = adj.ptr[w + 1]; col = adj.col; }
                    else {
                        if (!adj.dptr) break;
                        s0 = adj.dptr[w]; s1 = adj.dptr[w + 1]; col = adj.dcol;
                    }
#pragma unroll 1
                    for (uint32_t e0 = s0; e0 < s1; e0 += 32) {
                        const uint32_t ei = e0 + lane;
                        if (ei < s1) {
                            const uint32_t x = __ldg(col + ei);
                            const unsigned long long hit = fw & tgt_lookup(S, x);
                            if (hit) atomicOr(&S.done, hit);
                            const unsigned long long cand =
                                fw & ~hit & ~*(volatile unsigned long long *)&S.done;
                            if (cand) {
                                const int sl = tab_slot<DENSE>(T, x);
                                if (sl < 0) {
                                    S.overflow = 1;
                                } else {
                                    const unsigned long long old = atomicOr(&T.vis[sl], cand);
                                    const unsigned long long nw = cand & ~old;
                                    if (nw) {
                                        // pruning, queries.py:137-140
                                        unsigned long long pruned = 0;
                                        if (prune_dl || prune_bl) {
                                            const uint64_t *rx = rec + (size_t)x * rw;
                                            unsigned long long m = nw;
                                            while (m) {
                                                const int b = __ffsll((long long)m) - 1;
                                                m &= m - 1;
                                                bool p = false;
                                                if (prune_dl)
                                                    for (uint32_t k = 0; k < WDL; ++k)
                                                        p |= (dlo_u[b * WD + k] & __ldg(rx + k)) != 0;
                                                if (prune_bl && !p)
                                                    for (uint32_t k = 0; k < WBL; ++k)
                                                        p |= ((__ldg(rx + WDL + k) & ~bli_v[b * WBL + k]) |
                                                              (blo_v[b * WBL + k] & ~__ldg(rx + H + WDL + k))) != 0;
                                                if (p) pruned |= 1ull << b;
                                            }
                                        }
                                        const unsigned long long nx = nw & ~pruned;
                                        if (nx && atomicOr(&T.fr[nxt][sl], nx) == 0) {
                                            const uint32_t p = atomicAdd(&S.nlist[nxt], 1u);
                                            T.list[nxt][p] = (uint32_t)sl;
                                        }
                                    }
                                }
                            }
                        }
                        const unsigned long long act2 = S.active;
                        if ((*(volatile unsigned long long *)&S.done & act2) == act2) break;
                    }
                }
            }
            __syncthreads();
            if (tid == 0) S.nlist[cur] = 0;
            cur = nxt;
            __syncthreads();
        }
        __syncthreads();
        if (S.overflow) {
            if (!DENSE && tid == 0) {
                const uint32_t p = atomicAdd(&counters[CNT_OVERFLOW], 1u);
                ovf[p] = grp;
            }
        } else if (tid < (int)S.nq) {
            const uint32_t qi = S.qidx[tid];
            codes[qi] = ((S.done >> tid) & 1) ? DBL_BFS_POSITIVE : DBL_BFS_NEGATIVE;
            if (visited) visited[qi] = S.vcount[tid];
        }
        __syncthreads();
    }
}

static size_t bfs_smem(int wdl, int wbl, bool dense) {
    size_t s = (sizeof(BfsShared) + 15) & ~(size_t)15;
    s += (size_t)GQ * 8 * ((wdl > 0 ? wdl : 1) + 2 * wbl);
    if (!dense) s += (size_t)HCAP * (8 * 3 + 4 * 3);
    return s;
}

typedef void (*label_fn)(const uint64_t *, uint32_t, const uint32_t *, const uint32_t *, uint64_t,
                         uint32_t, uint8_t *, uint32_t *, uint32_t *, uint32_t *);

static label_fn pick_label(uint32_t wdl, uint32_t wbl) {
#define DBL_QK(A, B) if (wdl == A && wbl == B) return label_check_kernel<A, B>;
    DBL_QK(0, 1) DBL_QK(1, 1) DBL_QK(2, 1) DBL_QK(4, 1) DBL_QK(0, 2) DBL_QK(1, 2) DBL_QK(2, 2)
#undef DBL_QK
    return nullptr;
}

dbl_status run_query(const dbl_index *idx, dbl_graph *g, const uint32_t *u, const uint32_t *v,
                     uint64_t count, uint32_t flags, uint8_t *codes, uint32_t *visited) {
    if (count >= 0xffffffffull) { set_error("query batch too large"); return DBL_E_ARG; }
    if (idx->wdl > MAXW || idx->wbl > MAXW) {
        set_error("label width too large for the query kernels");
        return DBL_E_CONFIG;
    }
    const label_fn label = pick_label(idx->wdl, idx->wbl);
    dbl_status s;
    if ((s = g->q_pending.ensure(count * 8 + 64)) || (s = g->q_counters.ensure(CNT_WORDS * 4))) return s;
    uint32_t *pending = g->q_pending.as<uint32_t>();
    uint32_t *ovf = pending + count + 16;
    uint32_t *counters = g->q_counters.as<uint32_t>();
    DBL_CUDA(cudaMemsetAsync(counters, 0, CNT_WORDS * 4, g->stream));
    DBL_CUDA(cudaEventRecord(g->ev[2], g->stream));
    if (count) {
        int blocks = (int)((count + 255) / 256);
        if (blocks > g->sm_count * 16) blocks = g->sm_count * 16;
        if (label)
            label<<<blocks, 256, 0, g->stream>>>(idx->rec.as<uint64_t>(), idx->n, u, v, count, flags,
                                                   codes, visited, pending, counters);
        else
            label_check_generic<<<blocks, 256, 0, g->stream>>>(idx->rec.as<uint64_t>(), idx->n, idx->wdl,
                                                               idx->wbl, u, v, count, flags, codes, visited,
                                                               pending, counters);
        DBL_CHECK_LAUNCH("label_check_kernel");
    }
    DBL_CUDA(cudaEventRecord(g->ev[3], g->stream));
    if (count) {
        // K7 over the compacted pending list (persistent CTAs, group tickets)
        static int bps = -1;
        static size_t last_smem = 0;
        const size_t smem = bfs_smem(idx->wdl, idx->wbl, false);
        DBL_CUDA(cudaFuncSetAttribute((const void *)bfs_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (bps < 0 || last_smem != smem) {
            DBL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, bfs_kernel<false>, BFS_THREADS, smem));
            if (bps < 1) bps = 1;
            last_smem = smem;
        }
        Adj adj = graph_fwd(g);
        bfs_kernel<false><<<g->sm_count * bps, BFS_THREADS, smem, g->stream>>>(idx->rec.as<uint64_t>(), idx->wdl, idx->wbl, idx->n, adj,
                                                                  u, v, flags, pending, counters, ovf, codes,
                                                                  visited, nullptr);
        DBL_CHECK_LAUNCH("bfs_kernel");
        // dense re-run of overflowed groups: a few CTAs with n-sized slabs
        const size_t slab = (size_t)idx->n * 32;
        int dctas = 8;
        const size_t budget = (size_t)4 << 30;
        while (dctas > 1 && slab * dctas > budget) --dctas;
        if ((s = g->q_dense.ensure(slab * dctas + 16))) return s;
        const size_t dsmem = bfs_smem(idx->wdl, idx->wbl, true);
        DBL_CUDA(cudaFuncSetAttribute((const void *)bfs_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
        bfs_kernel<true><<<dctas, BFS_THREADS, dsmem, g->stream>>>(idx->rec.as<uint64_t>(), idx->wdl, idx->wbl, idx->n, adj, u, v,
                                                          flags, pending, counters, ovf, codes, visited,
                                                          g->q_dense.as<char>());
        DBL_CHECK_LAUNCH("bfs_kernel_dense");
    }
    DBL_CUDA(cudaEventRecord(g->ev[4], g->stream));
    return DBL_OK;
}

dbl_status query_finish(dbl_graph *g, uint32_t *err_out) {
    uint32_t h[CNT_WORDS];
    DBL_CUDA(cudaMemcpyAsync(h, g->q_counters.p, CNT_WORDS * 4, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    cudaEventElapsedTime(&g->t_label, g->ev[2], g->ev[3]);
    cudaEventElapsedTime(&g->t_bfs, g->ev[3], g->ev[4]);
    *err_out = h[CNT_ERR];
    return DBL_OK;
}

}  // namespace dbl
