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
#include <emmintrin.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "insert_one.cuh"

namespace dbl {

// Per-batch device counters.  Words [0, 8) are live during a batch and are
// left zeroed by the batch's last kernel, which first copies them to the
// result words [8, 16) (read by the host after the batch): no memset launch
// per batch.
enum { CNT_PENDING = 0, CNT_ERR = 1, CNT_TICKET = 2, CNT_OVERFLOW = 3, CNT_DTICKET = 4, CNT_TILE = 5,
       CNT_DONE = 6, CNT_WOVF = 7, CNT_WORDS = 8, CNT_RES = 8, CNT_ALL = 16 };
constexpr int GQ = 64;             // queries per BFS group
constexpr int HCAP = 2048;         // shared hash capacity (power of two)
constexpr int HBITS = 11;
constexpr int TCAP = 128;          // target table
constexpr int BFS_THREADS = 256;
constexpr uint32_t EMPTY = 0xffffffffu;
constexpr uint8_t UNRESOLVED = 0xff;

// Variant switches (build.build_variant -D flags; defaults = measured best)
#ifndef DBL_NO_PIVOT_PRUNE
#define DBL_NO_PIVOT_PRUNE 0   // 1: BFS fallbacks ignore the pivot sets
#endif
#ifndef DBL_LEAN_WAVES
#define DBL_LEAN_WAVES 1       // K6 grid cap in waves of resident CTAs
#endif
#ifndef DBL_LEAN_THREADS
#define DBL_LEAN_THREADS 256   // K6 CTA size
#endif
constexpr int LEAN_THREADS = DBL_LEAN_THREADS;
#ifndef DBL_DIGEST
#define DBL_DIGEST 1           // 0: query kernels never read the label digest
#endif
#ifndef DBL_DIGEST_REFRESH_MIN
#define DBL_DIGEST_REFRESH_MIN 65536   // smallest batch that recomputes a stale digest
#endif
#ifndef DBL_LEAN_WIDE
#define DBL_LEAN_WIDE 0        // 1: k > 64 also takes the lean gather (slower on cfg5)
#endif

// The build's pivot sets (reach_kernel): dmask = vertices reached from the
// pivot landmark h, scc = DL bits of the landmarks in h's SCC.  Every x in
// D(h) has those bits in dl_in[x], so for a query whose dl_out[u] meets scc
// the DL prune of queries.py:137-138 holds for every x in D(h); the BFS tests
// one bit of an L2-resident bitmap instead of reading x's record, before x
// takes a visited-table slot.  (Not stamping a pruned x changes nothing: it
// is pruned again on every visit and never expanded or counted.)  Inserts
// only grow D(h), so the stored subset stays sound; n = 0 disables it.
struct Pivot {
    const uint32_t *dmask;
    const unsigned long long *scc;
    uint32_t n;
    uint32_t pad;
};

// Per-call query arguments, passed by value to every query kernel.
struct QueryDesc {
    const uint32_t *u;
    const uint32_t *v;
    uint8_t *codes;
    uint32_t *visited;
    uint32_t count;
    uint32_t flags;
    int vec_ok;
    int pad;
    Pivot pv;
    uint32_t *hres;   // pinned host copy of the result words (written by the closing CTA), or nullptr
    const uint32_t *dig;   // label digest (n u32), or nullptr: every pair reads the full records
};

__device__ __forceinline__ bool in_pivot(const Pivot &pv, uint32_t x) {
    return x < pv.n && ((__ldg(pv.dmask + (x >> 5)) >> (x & 31)) & 1u);
}

// Does the query whose dl_out[u] is `dlo` (wdl words) take the pivot prune?
__device__ __forceinline__ bool pivot_query(const Pivot &pv, const unsigned long long *dlo, uint32_t wdl, bool prune_dl) {
    if (!prune_dl || pv.n == 0) return false;
    unsigned long long m = 0;
    for (uint32_t k = 0; k < wdl; ++k) m |= dlo[k] & __ldg(pv.scc + k);
    return m != 0;
}

__device__ __forceinline__ void ld_nc128(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}

// ------------------------------------------------------------ digest --
//
// One u32 per vertex x summarising its label record, so that most pairs are
// decided from an n x 4-byte table that stays in L2 (64 MB at n = 2^24,
// against 512 MB of records) and only the rest gather the two records:
//   bit 0   dl_out[x] has landmark 0 (exact)   bit 2   dl_in[x] has landmark 0
//   bit 1   dl_out[x] has any other landmark   bit 3   dl_in[x] has any other
//   4..17   bl_in[x] folded: bucket b -> bit 4 + (b % 64) % 14
//   18..31  bl_out[x] folded the same way
// Every decision it makes is one the full rules make (queries.py:102-108):
//   * landmark 0 in dl_out[u] and dl_in[v] is a witness of rule 1
//     (DL_POSITIVE);
//   * disjoint DL digests prove dl_out[u] & dl_in[v] == 0 (each digest bit
//     is the OR of a fixed set of label bits, the same sets for u and v), so
//     rule 1 does not fire, and a digest bit of u's folded bl_in missing from
//     v's proves a bucket in bl_in[u] \ bl_in[v] (likewise bl_out), so rule 2
//     fires (BL_NEGATIVE).
// Anything else is undecided and takes the record path, which applies the
// rules in order as before.  Landmark 0 is the pivot h, the top-scored
// landmark, so it witnesses almost every DL-positive pair on R-MAT graphs;
// measured on cfg2 / 2^22 uniform batches the digest decides 97.6% / 97.2%
// of the pairs (the 32-bit split 2 + 2 + 14 + 14 beat 4 + 4 + 12 + 12 and
// 3 + 3 + 13 + 13 by 0.2-1.8 points).
__device__ __forceinline__ uint32_t fold14(uint64_t x) {
    return (uint32_t)((x | (x >> 14) | (x >> 28) | (x >> 42) | (x >> 56)) & 0x3fffu);
}

__device__ __forceinline__ uint32_t digest_of(const uint64_t *__restrict__ r, uint32_t wdl, uint32_t wbl) {
    const uint32_t H = wdl + wbl;
    uint32_t d = 0;
    if (wdl) {
        const uint64_t in0 = __ldg(r), out0 = __ldg(r + H);
        uint64_t in_rest = in0 & ~1ull, out_rest = out0 & ~1ull;
        for (uint32_t k = 1; k < wdl; ++k) {
            in_rest |= __ldg(r + k);
            out_rest |= __ldg(r + H + k);
        }
        d = (uint32_t)(out0 & 1u) | (out_rest ? 2u : 0u) | ((uint32_t)(in0 & 1u) << 2) | (in_rest ? 8u : 0u);
    }
    uint32_t fi = 0, fo = 0;
    for (uint32_t k = 0; k < wbl; ++k) {
        fi |= fold14(__ldg(r + wdl + k));
        fo |= fold14(__ldg(r + H + wdl + k));
    }
    return d | (fi << 4) | (fo << 18);
}

__global__ void __launch_bounds__(256) digest_kernel(const uint64_t *__restrict__ rec, uint32_t n, uint32_t rs,
                                                     uint32_t wdl, uint32_t wbl, uint32_t *__restrict__ dig) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
        dig[x] = digest_of(rec + (size_t)x * rs, wdl, wbl);
}

// After an insert batch: recompute the digests of the vertices whose labels
// grew (the fixpoint's per-direction change bitmaps; seeds included).
__global__ void __launch_bounds__(256) digest_changed_kernel(const uint64_t *__restrict__ rec, uint32_t n,
                                                             uint32_t rs, uint32_t wdl, uint32_t wbl,
                                                             const uint32_t *__restrict__ bits0,
                                                             const uint32_t *__restrict__ bits1,
                                                             uint32_t *__restrict__ dig) {
    const uint32_t nw = (n + 31) / 32;
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
        uint32_t m = bits0[w] | bits1[w];
        while (m) {
            const uint32_t x = w * 32 + (uint32_t)(__ffs(m) - 1);
            m &= m - 1;
            if (x < n) dig[x] = digest_of(rec + (size_t)x * rs, wdl, wbl);
        }
    }
}

// Decide (u, v) from the digests: a code, or UNRESOLVED (read the records).
__device__ __forceinline__ uint8_t digest_decide(uint32_t du, uint32_t dv, bool use_dl, bool use_bl) {
    const uint32_t dl = du & (dv >> 2) & 3u;   // bit 0: landmark 0 common, bit 1: other DL bits may meet
    if (use_dl && (dl & 1u)) return DBL_DL_POSITIVE;
    const uint32_t fi_u = (du >> 4) & 0x3fffu, fi_v = (dv >> 4) & 0x3fffu;
    if (use_bl && (!use_dl || dl == 0) && ((fi_u & ~fi_v) | ((dv >> 18) & ~(du >> 18)))) return DBL_BL_NEGATIVE;
    return 0xff;
}

template <int WDL, int WBL>
__global__ void digest_kernel_t(const uint64_t *__restrict__ rec, uint32_t n, uint32_t *__restrict__ dig);

dbl_status digest_refresh(const dbl_index *idx, dbl_graph *g) {
    if (!DBL_DIGEST || idx->digest_version == idx->version) return DBL_OK;
    dbl_status s = idx->digest.ensure((size_t)idx->n * 4 + 16);
    if (s) return s;
    if (idx->n) {
        const uint32_t blocks = (idx->n + 255) / 256;
        const uint64_t *rec = idx->rec.as<uint64_t>();
        uint32_t *dig = idx->digest.as<uint32_t>();
        // one vertex per thread; the common widths load the record with
        // vector loads (templated), the rest word by word
#define DBL_DG(A, B) if (idx->wdl == A && idx->wbl == B) digest_kernel_t<A, B><<<blocks, 256, 0, g->stream>>>(rec, idx->n, dig); else
        DBL_DG(1, 1) DBL_DG(2, 1) DBL_DG(4, 1) DBL_DG(1, 2) DBL_DG(2, 2) DBL_DG(0, 1)
            digest_kernel<<<blocks < (uint32_t)g->sm_count * 8 ? blocks : g->sm_count * 8, 256, 0, g->stream>>>(
                rec, idx->n, idx->rs, idx->wdl, idx->wbl, dig);
#undef DBL_DG
        DBL_CHECK_LAUNCH("digest_kernel");
    }
    idx->digest_version = idx->version;
    return DBL_OK;
}

dbl_status digest_after_insert(dbl_index *idx, dbl_graph *g, bool was_current) {
    if (!DBL_DIGEST || !was_current) return DBL_OK;
    if (idx->n) {
        const size_t nw = ((size_t)idx->n + 31) / 32;
        if (g->changed_bits.bytes < nw * 8) return DBL_OK;   // no change bitmaps: stays stale
        uint32_t blocks = (uint32_t)((nw + 255) / 256);
        if (blocks > (uint32_t)g->sm_count * 4) blocks = g->sm_count * 4;
        const uint32_t *b0 = g->changed_bits.as<uint32_t>();
        digest_changed_kernel<<<blocks, 256, 0, g->stream>>>(idx->rec.as<uint64_t>(), idx->n, idx->rs, idx->wdl,
                                                             idx->wbl, b0, b0 + nw, idx->digest.as<uint32_t>());
        DBL_CHECK_LAUNCH("digest_changed_kernel");
    }
    idx->digest_version = idx->version;
    return DBL_OK;
}

// ------------------------------------------------------------------ K6 --

// runtime-width variant (any k, k')
__global__ void __launch_bounds__(256)
label_check_generic(const uint64_t *__restrict__ rec, uint32_t n, uint32_t wdl, uint32_t wbl,
                    const uint32_t *__restrict__ qu, const uint32_t *__restrict__ qv, uint64_t count,
                    uint32_t flags, uint8_t *__restrict__ codes, uint32_t *__restrict__ visited,
                    uint32_t *__restrict__ pending, uint32_t *__restrict__ counters) {
    const uint32_t H = wdl + wbl, RW = 2 * H, RS = rec_stride(H);
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
                const uint64_t *a = rec + (size_t)u * RS, *b = rec + (size_t)v * RS;
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
    unsigned long long dstart;   // done at the start of the current level (visited counts)
    unsigned long long active;
    unsigned long long sccq;   // queries taking the pivot prune
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
           const QueryDesc qd, const uint32_t *__restrict__ pending,
           uint32_t *__restrict__ counters, uint32_t *__restrict__ ovf, char *__restrict__ ws) {
    const uint32_t *__restrict__ qu = qd.u;
    const uint32_t *__restrict__ qv = qd.v;
    const uint32_t flags = qd.flags;
    uint8_t *__restrict__ codes = qd.codes;
    uint32_t *__restrict__ visited = qd.visited;
    const uint32_t H = WDL + WBL, rw = rec_stride(H);
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
            S.dstart = 0;
            S.sccq = 0;
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
            if (pivot_query(qd.pv, reinterpret_cast<const unsigned long long *>(ru + H), WDL, prune_dl))
                atomicOr(&S.sccq, 1ull << tid);
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
                    DBL_DCHECK(p < T.cap);
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
                    const unsigned long long raw = T.fr[cur][slot];
                    fw = raw & ~*(volatile unsigned long long *)&S.done;
                    T.fr[cur][slot] = 0;
                    // visited: every vertex of each level a query starts
                    // (levels 0..d-1 of a positive, all reached vertices of a
                    // negative), independent of the order within the level
                    unsigned long long m = raw & ~S.dstart;
                    while (m) {
                        const int b = __ffsll((long long)m) - 1;
                        m &= m - 1;
                        atomicAdd(&S.vcount[b], 1u);
                    }
                }
                fw = __shfl_sync(FULL, fw, 0);
                if (fw == 0) continue;
                const uint32_t w = tab_vertex<DENSE>(T, slot);
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
                            DBL_DCHECK(x < adj.n);
                            const unsigned long long hit = fw & tgt_lookup(S, x);
                            if (hit) atomicOr(&S.done, hit);
                            unsigned long long cand =
                                fw & ~hit & ~*(volatile unsigned long long *)&S.done;
                            if (cand & S.sccq && in_pivot(qd.pv, x)) cand &= ~S.sccq;
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
                                            DBL_DCHECK(p < T.cap);
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
            if (tid == 0) {
                S.nlist[cur] = 0;
                S.dstart = S.done;
            }
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

// ------------------------------------------------- per-warp BFS state --
//
// Bit-parallel pruned BFS of up to 32 queries on one warp (bit i of a 32-bit
// word = query i): frontier expansion is flattened across lanes (32 edges per
// step, the owner entry found by a shuffle search over the degree prefix),
// visited/frontier words live in a per-warp shared-memory hash table.  Used
// by the wide gather kernel (K6w) for its unresolved queries and by the
// tail-launched warp kernel (K7b).  A batch whose BFS outgrows the table is
// appended to an overflow list and finished by the 64-query group kernel
// (and, beyond that, the dense kernel).

#ifndef DBL_QMINB
#define DBL_QMINB 2
#endif
constexpr int WH = 128;            // per-warp BFS hash slots (power of two)
constexpr int WHBITS = 7;
constexpr int WT = 64;             // per-warp target table slots
constexpr int FUSED_THREADS = 256;

template <int WDL, int WBL>
struct WarpBfs {
    static constexpr int WD = WDL > 0 ? WDL : 1;
    uint32_t hkey[WH];
    uint32_t hvis[WH];
    uint32_t hfr[2][WH];
    uint16_t hlist[2][WH];
    uint32_t tkey[WT];
    uint32_t tmask[WT];
    uint32_t qidx[32];
    uint32_t qu[32];
    uint32_t qv[32];
    uint32_t vcnt[32];
    uint32_t nq;
    uint64_t qdlo[32 * WD];
    uint64_t qbli[32 * WBL];
    uint64_t qblo[32 * WBL];
    uint32_t nlist[2];
    uint32_t done;
    uint32_t overflow;
    uint32_t sccq;   // queries taking the pivot prune
};

// The 2H words of a record at p; 256-bit loads while 32-byte aligned
// (stride RS a multiple of 4 words), 128-bit ones for the rest.
template <int RW, int RS>
__device__ __forceinline__ void load_record(const uint64_t *p, uint64_t (&r)[RW]) {
    constexpr int V4 = RS % 4 == 0 ? RW / 4 * 4 : 0;
#pragma unroll
    for (int k = 0; k < V4; k += 4)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(r[k]), "=l"(r[k + 1]), "=l"(r[k + 2]), "=l"(r[k + 3]) : "l"(p + k));
#pragma unroll
    for (int k = V4; k < RW; k += 2)
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];"
                     : "=l"(r[k]), "=l"(r[k + 1]) : "l"(p + k));
}

template <int WDL, int WBL>
__global__ void __launch_bounds__(256) digest_kernel_t(const uint64_t *__restrict__ rec, uint32_t n,
                                                       uint32_t *__restrict__ dig) {
    constexpr int H = WDL + WBL, RW = 2 * H, RS = (int)rec_stride(H);
    const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    uint64_t r[RW];
    load_record<RW, RS>(rec + (size_t)x * RS, r);
    uint32_t d = 0;
    if (WDL) {
        uint64_t in_rest = r[0] & ~1ull, out_rest = r[H] & ~1ull;
#pragma unroll
        for (int k = 1; k < WDL; ++k) {
            in_rest |= r[k];
            out_rest |= r[H + k];
        }
        d = (uint32_t)(r[H] & 1u) | (out_rest ? 2u : 0u) | ((uint32_t)(r[0] & 1u) << 2) | (in_rest ? 8u : 0u);
    }
    uint32_t fi = 0, fo = 0;
#pragma unroll
    for (int k = 0; k < WBL; ++k) {
        fi |= fold14(r[WDL + k]);
        fo |= fold14(r[H + WDL + k]);
    }
    dig[x] = d | (fi << 4) | (fo << 18);
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t x, uint32_t &total) {
    const int lane = threadIdx.x & 31;
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += y;
    }
    total = __shfl_sync(FULL, v, 31);
    return v - x;
}

template <int WDL, int WBL>
__device__ __forceinline__ int wb_slot(WarpBfs<WDL, WBL> &B, uint32_t x) {
    uint32_t h = (x * 0x9E3779B1u) >> (32 - WHBITS);
#pragma unroll 1
    for (int probe = 0; probe < 32; ++probe) {
        const uint32_t k = B.hkey[h];
        if (k == x) return (int)h;
        if (k == EMPTY) {
            const uint32_t old = atomicCAS(&B.hkey[h], EMPTY, x);
            if (old == EMPTY || old == x) return (int)h;
        }
        h = (h + 1) & (WH - 1);
    }
    return -1;
}

template <int WDL, int WBL>
__device__ __forceinline__ uint32_t wb_target(const WarpBfs<WDL, WBL> &B, uint32_t x) {
    uint32_t h = (x * 0x9E3779B1u) >> 26;  // 6 bits
#pragma unroll 1
    for (int probe = 0; probe < WT; ++probe) {
        const uint32_t k = B.tkey[h];
        if (k == x) return B.tmask[h];
        if (k == EMPTY) return 0;
        h = (h + 1) & (WT - 1);
    }
    return 0;
}

// Bit-parallel pruned BFS for the nb (<= 32) queries staged in B (qidx, qu,
// qdlo, qbli, qblo, targets).  On return B.done holds the found bits and
// B.vcnt the per-query expansion counts; B.overflow is set if the table
// filled up (results then invalid).
template <int WDL, int WBL>
__device__ void warp_bfs(WarpBfs<WDL, WBL> &B, uint32_t nb, const uint64_t *__restrict__ rec,
                         const Adj &adj, bool prune_dl, bool prune_bl, const Pivot &pv) {
    constexpr int H = WDL + WBL, RW = 2 * H, RS = (int)rec_stride(H), WD = WarpBfs<WDL, WBL>::WD;
    const int lane = threadIdx.x & 31;
    const uint32_t all = nb == 32 ? FULL : ((1u << nb) - 1u);
    // sources
    if (lane < (int)nb) {
        const int sl = wb_slot(B, B.qu[lane]);
        if (sl < 0) {
            B.overflow = 1;
        } else {
            atomicOr(&B.hvis[sl], 1u << lane);
            if (atomicOr(&B.hfr[0][sl], 1u << lane) == 0) {
                const uint32_t p = atomicAdd(&B.nlist[0], 1u);
                B.hlist[0][p] = (uint16_t)sl;
            }
        }
    }
    __syncwarp();
    int cur = 0;
    for (;;) {
        const uint32_t ncur = *(volatile uint32_t *)&B.nlist[cur];
        const uint32_t dn = *(volatile uint32_t *)&B.done;
        if (ncur == 0 || (dn & all) == all || *(volatile uint32_t *)&B.overflow) break;
        const int nxt = cur ^ 1;
        for (uint32_t base = 0; base < ncur; base += 32) {
            // lane j takes frontier entry base + j
            const uint32_t ej = base + lane;
            uint32_t fw = 0, fc = 0, w = 0, b0 = 0, bl = 0, d0 = 0, dl = 0;
            if (ej < ncur) {
                const uint32_t sl = B.hlist[cur][ej];
                w = B.hkey[sl];
                const uint32_t raw = B.hfr[cur][sl];
                fw = raw & ~*(volatile uint32_t *)&B.done;
                fc = raw & ~dn;   // visited: the whole level for every query active at its start
                B.hfr[cur][sl] = 0;
                if (fw) {
                    b0 = __ldg(adj.ptr + w);
                    bl = __ldg(adj.ptr + w + 1) - b0;
                    if (adj.dptr) {
                        d0 = __ldg(adj.dptr + w);
                        dl = __ldg(adj.dptr + w + 1) - d0;
                    }
                }
            }
            // per-query expansion counts: lane q counts the entries holding bit q
            {
                for (int j = 0; j < 32; ++j) {
                    const uint32_t fj = __shfl_sync(FULL, fc, j);
                    if ((fj >> lane) & 1) B.vcnt[lane] += 1;
                }
            }
            uint32_t total = 0;
            const uint32_t excl = warp_excl_scan(bl + dl, total);
            for (uint32_t t0 = 0; t0 < total; t0 += 32) {
                const uint32_t t = t0 + lane;
                // owner: last lane with excl <= t (excl is non-decreasing)
                int k = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const uint32_t vv = __shfl_sync(FULL, excl, (k + st) & 31);
                    if (k + st < 32 && vv <= t) k += st;
                }
                // skip empty owners: excl equal for several lanes -> take the last
                const uint32_t ofw = __shfl_sync(FULL, fw, k);
                const uint32_t ob0 = __shfl_sync(FULL, b0, k), obl = __shfl_sync(FULL, bl, k);
                const uint32_t od0 = __shfl_sync(FULL, d0, k), oex = __shfl_sync(FULL, excl, k);
                if (t >= total) continue;
                const uint32_t r = t - oex;
                const uint32_t x = r < obl ? __ldg(adj.col + ob0 + r) : __ldg(adj.dcol + od0 + (r - obl));
                DBL_DCHECK(x < adj.n);
                const uint32_t hit = ofw & wb_target(B, x);
                if (hit) atomicOr(&B.done, hit);
                uint32_t cand = ofw & ~hit & ~*(volatile uint32_t *)&B.done;
                if (cand & B.sccq && in_pivot(pv, x)) cand &= ~B.sccq;
                if (!cand) continue;
                const int sl = wb_slot(B, x);
                if (sl < 0) { B.overflow = 1; continue; }
                const uint32_t old = atomicOr(&B.hvis[sl], cand);
                const uint32_t nw = cand & ~old;
                if (!nw) continue;
                uint32_t pruned = 0;
                if (prune_dl || prune_bl) {   // queries.py:137-140
                    uint64_t xr[RW];
                    load_record<RW, RS>(rec + (size_t)x * RS, xr);
                    uint32_t m = nw;
                    while (m) {
                        const int bq = __ffs(m) - 1;
                        m &= m - 1;
                        bool p = false;
                        if (prune_dl) {
#pragma unroll
                            for (int q = 0; q < WDL; ++q) p |= (B.qdlo[bq * WD + q] & xr[q]) != 0;
                        }
                        if (prune_bl && !p) {
#pragma unroll
                            for (int q = 0; q < WBL; ++q)
                                p |= ((xr[WDL + q] & ~B.qbli[bq * WBL + q]) | (B.qblo[bq * WBL + q] & ~xr[H + WDL + q])) != 0;
                        }
                        if (p) pruned |= 1u << bq;
                    }
                }
                const uint32_t nx = nw & ~pruned;
                if (nx && atomicOr(&B.hfr[nxt][sl], nx) == 0) {
                    const uint32_t p = atomicAdd(&B.nlist[nxt], 1u);
                    DBL_DCHECK(p < (uint32_t)WH);
                    B.hlist[nxt][p] = (uint16_t)sl;
                }
            }
            __syncwarp();
        }
        __syncwarp();
        if (lane == 0) B.nlist[cur] = 0;
        cur = nxt;
        __syncwarp();
    }
    __syncwarp();
}

// Run the warp's staged batch (B.nq queries) and write its answers.
#ifdef DBL_BFS_NOINLINE
#define DBL_BFS_INLINE __noinline__
#else
#define DBL_BFS_INLINE
#endif
template <int WDL, int WBL>
__device__ DBL_BFS_INLINE void warp_bfs_batch(WarpBfs<WDL, WBL> &B, const uint64_t *__restrict__ rec, const Adj &adj,
                               bool prune_dl, bool prune_bl, const Pivot &pv, uint8_t *__restrict__ codes,
                               uint32_t *__restrict__ visited, uint32_t *__restrict__ ovf_list,
                               uint32_t *__restrict__ counters, int ovf_counter) {
    const int lane = threadIdx.x & 31;
    const uint32_t nb = B.nq;
    for (int i = lane; i < WH; i += 32) {
        B.hkey[i] = EMPTY; B.hvis[i] = 0; B.hfr[0][i] = 0; B.hfr[1][i] = 0;
    }
    for (int i = lane; i < WT; i += 32) { B.tkey[i] = EMPTY; B.tmask[i] = 0; }
    B.vcnt[lane] = 0;
    if (lane == 0) { B.nlist[0] = 0; B.nlist[1] = 0; B.done = 0; B.overflow = 0; }
    __syncwarp();
    if (lane < (int)nb) {  // target table: v -> bit lane
        const uint32_t v = B.qv[lane];
        uint32_t h = (v * 0x9E3779B1u) >> 26;
        for (;;) {
            const uint32_t old = atomicCAS(&B.tkey[h], EMPTY, v);
            if (old == EMPTY || old == v) { atomicOr(&B.tmask[h], 1u << lane); break; }
            h = (h + 1) & (WT - 1);
        }
    }
    {
        const bool sq = lane < (int)nb &&
                        pivot_query(pv, reinterpret_cast<const unsigned long long *>(&B.qdlo[lane * WarpBfs<WDL, WBL>::WD]),
                                    WDL, prune_dl);
        const uint32_t m = __ballot_sync(FULL, sq);
        if (lane == 0) B.sccq = m;
    }
    __syncwarp();
    warp_bfs<WDL, WBL>(B, nb, rec, adj, prune_dl, prune_bl, pv);
    const bool ovf = B.overflow != 0;
    const uint32_t dn = B.done;
    if (lane < (int)nb) {
        const uint32_t qi = B.qidx[lane];
        if (ovf) {  // hand the batch to the group kernels via an overflow list
            const uint32_t p = atomicAdd(&counters[ovf_counter], 1u);
            ovf_list[p] = qi;
        } else {
            codes[qi] = ((dn >> lane) & 1) ? DBL_BFS_POSITIVE : DBL_BFS_NEGATIVE;
            if (visited) visited[qi] = B.vcnt[lane];
        }
    }
    __syncwarp();
    if (lane == 0) B.nq = 0;
    __syncwarp();
}

// Close a batch: publish the live counters to the result words and zero them
// for the next batch (stream order makes this the batch's last access).
// The batch's last CTA moves the live counters to the result words (and to
// the caller-visible pinned copy, so the host reads them after its stream
// sync without a device->host copy) and zeroes them for the next batch.
__device__ __forceinline__ void close_batch(uint32_t *counters, uint32_t *hres) {
#pragma unroll
    for (int i = 0; i < CNT_WORDS; ++i) {
        const uint32_t c = counters[i];
        counters[CNT_RES + i] = c;
        if (hres) hres[i] = c;
        counters[i] = 0;
    }
    // (no system fence: the host reads hres only after the stream sync, and
    // kernel completion makes the pinned writes visible)
}

__global__ void finish_batch_kernel(uint32_t *__restrict__ counters, uint32_t *hres) {
    if (threadIdx.x == 0) close_batch(counters, hres);
}

// Launch geometry of the hard path, handed to the fused kernel so that its
// last CTA can tail-launch the group and dense kernels when (and only when)
// a warp's BFS table overflowed.
struct HardArgs {
    int grid, dctas;
    uint32_t smem, dsmem;
    uint32_t wdl, wbl;
    uint32_t *ovf;
    char *ws;
    int wgrid;          // warp-BFS kernel (lean path)
    uint32_t wsmem;
    uint32_t *wovf;
};

// ------------------------------------------------- K6 wide: quad gathers --
//
// Records wider than 32 bytes (k > 64) live at 64/128-byte strides.  Random
// gathers that miss L2 are bound by L1->L2 requests, not bytes (measured with
// tools/ubench_gather: ~37 G requests/s whether a request carries one sector
// or a whole 128-byte line), and a thread reading its own 80-byte record
// issues three requests (32 + 32 + 16 bytes).  Here a lane quad reads one
// record: lane j of the quad loads 32-byte chunk j, so one warp instruction
// fetches 8 records with one request per record.  A warp tile is 32 queries
// gathered in 4 rounds of 8 (u and v chunks, all 8 loads in flight), the
// rules are evaluated inside each quad (the dl_out words a lane needs come
// from the quad lane holding them, by shuffle; the BL words of u and v sit in
// the same lane), and the codes move to lane 8r + i.  Unresolved queries are
// staged for the warp's bit-parallel BFS straight from the lanes holding the
// words.
__device__ __forceinline__ uint64_t shfl64(uint64_t x, int src) {
    const uint32_t lo = __shfl_sync(FULL, (uint32_t)x, src), hi = __shfl_sync(FULL, (uint32_t)(x >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

#ifndef DBL_QUAD_DEFER
#define DBL_QUAD_DEFER 1
#endif
template <int WDL, int WBL>
__global__ void __launch_bounds__(FUSED_THREADS, DBL_QMINB)
query_quad_kernel(const uint64_t *__restrict__ rec, uint32_t n, Adj adj, const QueryDesc qd,
                  uint32_t *__restrict__ pending, uint32_t *__restrict__ counters, const HardArgs ha) {
    constexpr int H = WDL + WBL, RW = 2 * H, RS = (int)rec_stride(H), WD = WarpBfs<WDL, WBL>::WD;
    constexpr int C = (RW + 3) / 4;   // 32-byte chunks per record
    static_assert(RS % 4 == 0 && C <= 4, "quad gather: 32-byte aligned records of at most 128 bytes");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int qi = lane >> 2, qj = lane & 3, qbase = lane & ~3;
    WarpBfs<WDL, WBL> &B = reinterpret_cast<WarpBfs<WDL, WBL> *>(smem_raw)[wid];
    const uint32_t count = qd.count, flags = qd.flags;
    const bool use_dl = flags & DBL_F_USE_DL, use_bl = flags & DBL_F_USE_BL;
    const bool thm1 = use_dl && (flags & DBL_F_THM1), thm2 = use_dl && (flags & DBL_F_THM2);
    const bool prune_dl = use_dl && (flags & DBL_F_PRUNE_DL), prune_bl = use_bl && (flags & DBL_F_PRUNE_BL);
    if (lane == 0) B.nq = 0;
    __syncwarp();
    for (;;) {
        uint32_t tile = 0;
        if (lane == 0) tile = atomicAdd(&counters[CNT_TILE], 1u);
        tile = __shfl_sync(FULL, tile, 0);
        const uint64_t q0 = (uint64_t)tile * 32;
        if (q0 >= count) break;
        const uint64_t q = q0 + lane;
        const bool inb = q < count;
        uint32_t u = 0, v = 0;
        if (inb) { u = __ldg(qd.u + q); v = __ldg(qd.v + q); }
        const bool bad = inb && (u >= n || v >= n);
        const bool live = inb && !bad && u != v;
        // pairs the digest decides skip the record gather
        uint32_t dcode = UNRESOLVED;
        if (qd.dig && live) dcode = digest_decide(__ldg(qd.dig + u), __ldg(qd.dig + v), use_dl, use_bl);
        const bool need = live && dcode == UNRESOLVED;
        // gather: round r, quad i -> query 8r + i, lane j -> chunk j
        uint64_t cu[4][4], cv[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int src = 8 * r + qi;
            const uint32_t su = __shfl_sync(FULL, u, src), sv = __shfl_sync(FULL, v, src);
            const bool sl = __shfl_sync(FULL, (int)need, src) != 0;
            if (sl && qj < C) {
                const uint64_t *pu = rec + (size_t)su * RS + 4 * qj, *pv = rec + (size_t)sv * RS + 4 * qj;
                asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                             : "=l"(cu[r][0]), "=l"(cu[r][1]), "=l"(cu[r][2]), "=l"(cu[r][3]) : "l"(pu));
                asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                             : "=l"(cv[r][0]), "=l"(cv[r][1]), "=l"(cv[r][2]), "=l"(cv[r][3]) : "l"(pv));
            } else {
#pragma unroll
                for (int t = 0; t < 4; ++t) cu[r][t] = cv[r][t] = 0;
            }
        }
        // rules 1-4 per quad (queries.py:96-114); lane j holds record words 4j..4j+3
        uint32_t mycode = UNRESOLVED;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            uint64_t r1 = 0, r2 = 0, r3 = 0, r4 = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int w = 4 * qj + t;
                if (WDL > 0) {
                    // out-half DL word k = w is record word H + k: quad lane (H + w) / 4, slot (H + t) % 4
                    const int srcl = (qbase + ((H + 4 * qj + t) >> 2)) & 31;
                    const uint64_t ou = shfl64(cu[r][(H + t) & 3], srcl), ov = shfl64(cv[r][(H + t) & 3], srcl);
                    if (w < WDL) {
                        r1 |= ou & cv[r][t];                               // dl_out[u] & dl_in[v]
                        r3 |= ov & cu[r][t];                               // dl_out[v] & dl_in[u]
                        r4 |= (ou & cu[r][t]) | (ov & cv[r][t]);           // Theorem 2
                    }
                }
                if (w >= WDL && w < H) r2 |= cu[r][t] & ~cv[r][t];         // bl_in[u] \ bl_in[v]
                if (w >= H + WDL && w < RW) r2 |= cv[r][t] & ~cu[r][t];    // bl_out[v] \ bl_out[u]
            }
            uint32_t bits = (r1 != 0) | ((r2 != 0) << 1) | ((r3 != 0) << 2) | ((r4 != 0) << 3);
            bits |= __shfl_xor_sync(FULL, bits, 1);
            bits |= __shfl_xor_sync(FULL, bits, 2);
            uint32_t c = UNRESOLVED;
            if (use_dl && (bits & 1)) c = DBL_DL_POSITIVE;
            else if (use_bl && (bits & 2)) c = DBL_BL_NEGATIVE;
            else if (thm1 && (bits & 4)) c = DBL_THM1_NEGATIVE;
            else if (thm2 && (bits & 8)) c = DBL_THM2_NEGATIVE;
            const uint32_t cc = __shfl_sync(FULL, c, (lane & 7) << 2);
            if ((lane >> 3) == r) mycode = cc;
        }
        uint32_t code = dcode != UNRESOLVED ? dcode : mycode;
        if (bad) {
            atomicOr(&counters[CNT_ERR], 1u);
            code = 0xfe;
        } else if (inb && u == v) {
            code = DBL_REFLEXIVE;
        }
        const bool unres = live && code == UNRESOLVED;
        if (inb && !unres) {
            qd.codes[q] = (uint8_t)code;
            if (qd.visited) qd.visited[q] = 0;
        }
        const uint32_t mask = __ballot_sync(FULL, unres);
        if (mask) {
            // stage the unresolved queries; the bit-parallel BFS runs once 32
            // have accumulated (and after the last tile): on cfg5 ~17% of
            // tiles hold one, and a BFS of 1 query costs the warp the same
            // latency chain as one of 32
            uint32_t nq0 = B.nq;
            if (nq0 + __popc(mask) > 32) {
                warp_bfs_batch<WDL, WBL>(B, rec, adj, prune_dl, prune_bl, qd.pv, qd.codes, qd.visited, pending,
                                         counters, CNT_PENDING);
                nq0 = 0;
            }
            if (unres) {
                const uint32_t slot = nq0 + __popc(mask & ((1u << lane) - 1u));
                B.qidx[slot] = (uint32_t)q;
                B.qu[slot] = u;
                B.qv[slot] = v;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int lq = 8 * r + qi;
                if (!((mask >> lq) & 1u)) continue;
                const uint32_t slot = nq0 + __popc(mask & ((1u << lq) - 1u));
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int w = 4 * qj + t;
                    if (w >= H && w < H + WDL) B.qdlo[slot * WD + (w - H)] = cu[r][t];
                    if (w >= WDL && w < H) B.qbli[slot * WBL + (w - WDL)] = cv[r][t];
                    if (w >= H + WDL && w < RW) B.qblo[slot * WBL + (w - H - WDL)] = cv[r][t];
                }
            }
            __syncwarp();
            if (lane == 0) B.nq = nq0 + __popc(mask);
            __syncwarp();
#if !DBL_QUAD_DEFER
            warp_bfs_batch<WDL, WBL>(B, rec, adj, prune_dl, prune_bl, qd.pv, qd.codes, qd.visited, pending, counters,
                                     CNT_PENDING);
            __syncwarp();
#endif
        }
    }
    __syncwarp();
    if (B.nq)
        warp_bfs_batch<WDL, WBL>(B, rec, adj, prune_dl, prune_bl, qd.pv, qd.codes, qd.visited, pending, counters,
                                 CNT_PENDING);
    // the last CTA out closes the batch, or tail-launches the group/dense
    // kernels for BFS batches that outgrew the warp tables
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(&counters[CNT_DONE], 1u);
        if (prev == gridDim.x - 1) {
            __threadfence();
            const uint32_t npend = *(volatile uint32_t *)&counters[CNT_PENDING];
            if (npend == 0) {
                close_batch(counters, qd.hres);
            } else {
                bfs_kernel<false><<<ha.grid, BFS_THREADS, ha.smem, cudaStreamTailLaunch>>>(
                    rec, ha.wdl, ha.wbl, n, adj, qd, pending, counters, ha.ovf, nullptr);
                if (ha.ws)
                    bfs_kernel<true><<<ha.dctas, BFS_THREADS, ha.dsmem, cudaStreamTailLaunch>>>(
                        rec, ha.wdl, ha.wbl, n, adj, qd, pending, counters, ha.ovf, ha.ws);
                finish_batch_kernel<<<1, 32, 0, cudaStreamTailLaunch>>>(counters, qd.hres);
            }
        }
    }
}

// ------------------------------------------------ K6 lean + K7 warp BFS --
//
// The throughput path.  K6 is the leanest possible gather: one query per
// thread per grid-stride step, both endpoints' records fetched with one
// 256-bit read-only load each, rules 0-4, the code (and visited = 0) stored,
// unresolved queries appended to the pending list with one warp-aggregated
// atomic.  No shared memory and few registers, so 2048 threads per SM keep
// ~4k record sectors in flight (measured: a one-query-per-thread gather beats
// persistent multi-query tiles by ~30% on 1M queries).
//
// K7a: the queries the label rules leave open (0.5% on R-MAT) are queued per
// CTA and answered by warp_query_bfs -- a pruned BFS of one query by one
// warp, bounded to TB_Q expanded vertices (on R-MAT the fallback visits <= 3)
// -- on a dedicated BFS warp while the other warps still gather.  A query
// that outgrows the bounds goes to the pending list, which the last CTA
// hands to the tail-launched warp kernel (K7b: bit-parallel BFS of <= 32
// queries per warp), and beyond that to the 64-query group and dense kernels.
// The answer equals the reference's: pruning only removes vertices that
// cannot reach v (a pruned x reaching v would give dl_out[u] & dl_in[v] != 0
// or violate BL containment), so v is found iff it is reachable, in any
// visiting order.
constexpr int TB_Q = 8;
constexpr uint32_t DQ_CAP = 128;   // deferred queries per CTA (more go to the warp BFS)
// A deferred query: its index, endpoints and the words its pruning needs
// (dl_out[u], bl_in[v], bl_out[v]; queries.py:137-140).
template <int WDL, int WBL>
struct DeferQ {
    static constexpr int WD = WDL > 0 ? WDL : 1;
    uint64_t dlo[DQ_CAP][WD], bli[DQ_CAP][WBL], blo[DQ_CAP][WBL];
    uint32_t i[DQ_CAP], u[DQ_CAP], v[DQ_CAP];
    uint32_t n;             // slots claimed (may exceed DQ_CAP: the rest go to the pending list)
};
#ifndef DBL_LMINB
#define DBL_LMINB 8
#endif

// The same bounded pruned BFS with the 32 lanes of a warp on one query: a
// frontier vertex's adjacency is read 32 neighbours at a time and their
// pruning words are gathered in parallel, so a level costs about two memory
// round trips instead of one per 4 neighbours.  The expanded/visited list
// (<= TB_Q) lives in the warp's slot of `wq`.  Warp-uniform result; TB_EW
// bounds the neighbours of one expanded vertex.
constexpr uint32_t TB_EW = 256;

template <int WDL, int WBL>
__device__ __forceinline__ int warp_query_bfs(const uint64_t *__restrict__ rec, const Adj &adj, uint32_t u, uint32_t v,
                                              const uint64_t *dlo_u, const uint64_t *bli_v, const uint64_t *blo_v,
                                              bool prune_dl, bool prune_bl, const Pivot &pv, uint32_t *wq,
                                              uint32_t *vcount) {
    const bool sq = pivot_query(pv, reinterpret_cast<const unsigned long long *>(dlo_u), WDL, prune_dl);
    constexpr int H = WDL + WBL, RW = 2 * H, RS = (int)rec_stride(H);
    const int lane = threadIdx.x & 31;
    if (lane == 0) wq[0] = u;
    __syncwarp();
    uint32_t qn = 1, lvl_end = 1;   // wq[0, lvl_end): the levels up to the one being expanded
    for (uint32_t head = 0; head < qn; ++head) {
        if (head == lvl_end) lvl_end = qn;
        const uint32_t w = wq[head];
        *vcount = lvl_end;
        for (int seg = 0; seg < 2; ++seg) {
            const uint32_t *ptr = seg ? adj.dptr : adj.ptr;
            if (!ptr) break;
            const uint32_t *col = seg ? adj.dcol : adj.col;
            const uint32_t s0 = __ldg(ptr + w), s1 = __ldg(ptr + w + 1);
            if (s1 - s0 > TB_EW) return 2;
            for (uint32_t j0 = s0; j0 < s1; j0 += 32) {
                const uint32_t j = j0 + lane;
                const bool ok = j < s1;
                const uint32_t x = ok ? __ldg(col + j) : 0xffffffffu;
                DBL_DCHECK(!ok || x < adj.n);
                if (__any_sync(FULL, ok && x == v)) return 1;   // target test precedes the visited test
                bool keep = ok;
                for (uint32_t k = 0; k < qn; ++k) keep &= wq[k] != x;
                if (keep && sq && in_pivot(pv, x)) keep = false;   // pruned
                if (keep && (prune_dl || prune_bl)) {
                    const uint64_t *rx = rec + (size_t)x * RS;
                    bool p = false;
                    if (prune_dl) {   // queries.py:137-138
#pragma unroll
                        for (int k = 0; k < WDL; ++k) p |= (dlo_u[k] & __ldg(rx + k)) != 0;
                    }
                    if (prune_bl && !p) {   // queries.py:139-140
#pragma unroll
                        for (int k = 0; k < WBL; ++k)
                            p |= ((__ldg(rx + WDL + k) & ~bli_v[k]) | (blo_v[k] & ~__ldg(rx + H + WDL + k))) != 0;
                    }
                    keep = !p;
                }
                const unsigned m = __ballot_sync(FULL, keep);
                if (!m) continue;
                if (qn + __popc(m) > TB_Q) return 2;
                __syncwarp();
                if (keep) wq[qn + __popc(m & ((1u << lane) - 1u))] = x;
                __syncwarp();
                qn += __popc(m);
            }
        }
    }
    *vcount = qn;
    return 0;
}

template <int WDL, int WBL>
__global__ void bfs_warp_kernel(const uint64_t *__restrict__ rec, uint32_t n, Adj adj, const QueryDesc qd,
                                uint32_t *__restrict__ pending, uint32_t *__restrict__ wovf,
                                uint32_t *__restrict__ counters, const HardArgs ha);

#ifndef DBL_LMINB_WIDE
#define DBL_LMINB_WIDE 4
#endif
#ifndef DBL_TBFS_ALL
#define DBL_TBFS_ALL 0
#endif
#ifndef DBL_EXP_NOBFS
#define DBL_EXP_NOBFS 0   // experiment builds only: skip the deferred BFS (answers incomplete)
#endif
constexpr uint8_t QUEUED = 0xfc;   // in the CTA's BFS queue (code written later)
#ifndef DBL_QPT_HOST
#define DBL_QPT_HOST 4   // pairs per thread per step when they are read over PCIe (4 or 8)
#endif
#ifndef DBL_QPT_DEV
#define DBL_QPT_DEV 0    // 1: device-resident pairs take the DBL_QPT_HOST kernel too
#endif
#ifndef DBL_QPT_DPRE
#define DBL_QPT_DPRE 1   // multi-pair kernel: every digest load of a thread's pairs issued first
#endif
#ifndef DBL_QPT_MINB
#define DBL_QPT_MINB 4   // resident 256-thread CTAs per SM of the multi-pair kernel
#endif

// Rules 0-4 for pair i = (u, v) (queries.py:94-114).  Returns the code, or
// QUEUED if the query went to the CTA's BFS queue, or UNRESOLVED if it is
// open and the queue is full (the caller appends it to the pending list).
template <int WDL, int WBL, bool TBFS>
__device__ __forceinline__ uint8_t lean_eval(const uint64_t *__restrict__ rec, const uint32_t *__restrict__ dig,
                                             uint32_t n, const Adj &adj, uint32_t i,
                                             uint32_t u, uint32_t v, bool use_dl, bool use_bl, bool thm1, bool thm2,
                                             DeferQ<WDL, WBL> &dq, uint32_t *__restrict__ counters,
                                             uint32_t du = 0, uint32_t dv = 0, bool dpre = false) {
    constexpr int H = WDL + WBL, RW = 2 * H, RS = (int)rec_stride(H);
    if (u >= n || v >= n) {
        atomicOr(&counters[CNT_ERR], 1u);
        return 0xfe;
    }
    if (u == v) return DBL_REFLEXIVE;
    if (dig) {
        // dpre: the caller loaded both digest words ahead (all of its pairs'
        // loads in flight at once)
        const uint8_t c = dpre ? digest_decide(du, dv, use_dl, use_bl)
                               : digest_decide(__ldg(dig + u), __ldg(dig + v), use_dl, use_bl);
        if (c != 0xff) return c;
    }
    uint64_t a[RW], b[RW];
    load_record<RW, RS>(rec + (size_t)u * RS, a);
    load_record<RW, RS>(rec + (size_t)v * RS, b);
    uint64_t r1 = 0, r2 = 0, r3 = 0, r4 = 0;
#pragma unroll
    for (int k = 0; k < WDL; ++k) {
        r1 |= a[H + k] & b[k];             // dl_out[u] & dl_in[v]
        r3 |= b[H + k] & a[k];             // dl_out[v] & dl_in[u]
        r4 |= (a[H + k] & a[k]) | (b[H + k] & b[k]);
    }
#pragma unroll
    for (int k = 0; k < WBL; ++k)
        r2 |= (a[WDL + k] & ~b[WDL + k]) | (b[H + WDL + k] & ~a[H + WDL + k]);
    if (use_dl && r1) return DBL_DL_POSITIVE;
    if (use_bl && r2) return DBL_BL_NEGATIVE;
    if (thm1 && r3) return DBL_THM1_NEGATIVE;
    if (thm2 && r4) return DBL_THM2_NEGATIVE;
    if (TBFS) {
        const uint32_t slot = atomicAdd(&dq.n, 1u);
        if (slot < DQ_CAP) {
            dq.i[slot] = i;
            dq.u[slot] = u;
            dq.v[slot] = v;
#pragma unroll
            for (int k = 0; k < WDL; ++k) dq.dlo[slot][k] = a[H + k];   // still in registers
#pragma unroll
            for (int k = 0; k < WBL; ++k) {
                dq.bli[slot][k] = b[WDL + k];
                dq.blo[slot][k] = b[H + WDL + k];
            }
            asm volatile("prefetch.global.L2 [%0];" ::"l"(adj.ptr + u));
            return QUEUED;
        }
    }
    return UNRESOLVED;
}

// Open queries of one warp step (unres lanes) go to the global pending list
// with one warp-aggregated atomic.
__device__ __forceinline__ void lean_pend(bool unres, uint32_t i, uint32_t *__restrict__ pending,
                                          uint32_t *__restrict__ counters) {
    const int lane = threadIdx.x & 31;
    const unsigned m = __ballot_sync(FULL, unres);
    if (m) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&counters[CNT_PENDING], (uint32_t)__popc(m));
        base = __shfl_sync(FULL, base, 0);
        if (unres) pending[base + __popc(m & ((1u << lane) - 1u))] = i;
    }
}

// QPT = 1: device-resident pairs, one query per thread per step.
// QPT = 4: pairs read from pinned host memory over PCIe (zero-copy): a
// thread takes 4 consecutive pairs with one 16-byte load of u and of v, so a
// warp instruction asks PCIe for 512 contiguous bytes instead of 128, and
// writes their 4 codes with one store; PCIe, not the gather, bounds it.
// 8 CTAs/SM (32 registers) for the 32-byte records of k <= 64; wide records
// (2 x 80 bytes at k = 256) spill at that cap, so they trade occupancy for
// registers
template <int WDL, int WBL, int QPT>
__global__ void __launch_bounds__(LEAN_THREADS, (QPT > 1 ? DBL_QPT_MINB : (WDL + WBL <= 3 ? DBL_LMINB : DBL_LMINB_WIDE)) * 256 / LEAN_THREADS)
label_lean_kernel(const uint64_t *__restrict__ rec, uint32_t n, const Adj adj, const QueryDesc qd,
                  uint32_t *__restrict__ pending, uint32_t *__restrict__ counters, const HardArgs ha) {
    // the per-thread BFS pays off for k <= 64; with wider labels (cfg5:
    // k = 256, d = 16) most fallbacks outgrow its bounds (measured: 79% of
    // cfg5's unresolved queries), so they go straight to the warp BFS
    constexpr bool TBFS = DBL_TBFS_ALL || WDL <= 1;
    const uint32_t flags = qd.flags, count = qd.count;
    const bool use_dl = flags & DBL_F_USE_DL, use_bl = flags & DBL_F_USE_BL;
    const bool thm1 = use_dl && (flags & DBL_F_THM1), thm2 = use_dl && (flags & DBL_F_THM2);
    const bool prune_dl = use_dl && (flags & DBL_F_PRUNE_DL), prune_bl = use_bl && (flags & DBL_F_PRUNE_BL);
    const int lane = threadIdx.x & 31;
    // Unresolved queries are deferred to a per-CTA queue (their BFS inputs
    // staged in shared memory, the source's row pointer prefetched into L2),
    // so a BFS never stalls the gathers (measured alternatives, DESIGN.md §4:
    // a dedicated BFS warp per CTA overlapping the gathers, 25.8 vs 23.1 us
    // -- the gathers lose a warp's worth of requests in flight).
    const int wid = threadIdx.x >> 5;
    __shared__ DeferQ<WDL, WBL> dq;
    if (threadIdx.x == 0) dq.n = 0;
    __syncthreads();
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x;
    if constexpr (QPT == 1) {
        const uint32_t cr = (count + 31) & ~31u;
        // the next iteration's pair is loaded while this one's records are in
        // flight (one dependent round trip per iteration instead of two)
        uint32_t nu = 0, nv = 0;
        if (i0 < count) { nu = __ldg(qd.u + i0); nv = __ldg(qd.v + i0); }
        for (uint32_t i = i0; i < cr; i += stride) {
            bool unres = false;
            const uint32_t u = nu, v = nv;
            const uint32_t inext = i + stride;
            if (inext < count) { nu = __ldg(qd.u + inext); nv = __ldg(qd.v + inext); }
            if (i < count) {
                const uint8_t code = lean_eval<WDL, WBL, TBFS>(rec, qd.dig, n, adj, i, u, v, use_dl, use_bl, thm1, thm2, dq,
                                                               counters);
                if (code != QUEUED) {
                    qd.codes[i] = code;
                    if (qd.visited) qd.visited[i] = 0;
                    unres = code == UNRESOLVED;
                }
            }
            lean_pend(unres, i, pending, counters);
        }
    } else {
        // (run_query takes this path only for 16-byte aligned u, v and
        // 4-byte aligned codes / 16-byte aligned visited)
        const uint32_t nblk = (count + QPT - 1) / QPT, cr = (nblk + 31) & ~31u;
        for (uint32_t bi = i0; bi < cr; bi += stride) {
            const uint32_t q0 = bi * QPT;
            uint32_t us[QPT], vs[QPT];
            const bool full = q0 + QPT <= count;
            if (bi < nblk) {
                if (full) {
#pragma unroll
                    for (int c = 0; c < QPT / 4; ++c) {
                        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(qd.u + q0) + c);
                        const uint4 b = __ldg(reinterpret_cast<const uint4 *>(qd.v + q0) + c);
                        us[4 * c] = a.x; us[4 * c + 1] = a.y; us[4 * c + 2] = a.z; us[4 * c + 3] = a.w;
                        vs[4 * c] = b.x; vs[4 * c + 1] = b.y; vs[4 * c + 2] = b.z; vs[4 * c + 3] = b.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < QPT; ++j) {
                        us[j] = q0 + j < count ? __ldg(qd.u + q0 + j) : 0;
                        vs[j] = q0 + j < count ? __ldg(qd.v + q0 + j) : 0;
                    }
                }
            }
            uint8_t cs[QPT];
            uint32_t dus[QPT], dvs[QPT];
            if (DBL_QPT_DPRE && qd.dig) {
#pragma unroll
                for (int j = 0; j < QPT; ++j) {
                    dus[j] = bi < nblk && us[j] < n ? __ldg(qd.dig + us[j]) : 0;
                    dvs[j] = bi < nblk && vs[j] < n ? __ldg(qd.dig + vs[j]) : 0;
                }
            }
#pragma unroll
            for (int j = 0; j < QPT; ++j) {
                bool unres = false;
                cs[j] = QUEUED;
                if (bi < nblk && q0 + j < count) {
                    cs[j] = lean_eval<WDL, WBL, TBFS>(rec, qd.dig, n, adj, q0 + j, us[j], vs[j], use_dl, use_bl, thm1, thm2,
                                                      dq, counters, dus[j], dvs[j], DBL_QPT_DPRE);
                    unres = cs[j] == UNRESOLVED;
                }
                lean_pend(unres, q0 + j, pending, counters);
            }
            if (bi < nblk) {
                // queued codes are written by the BFS later: store the others
                bool anyq = false;
#pragma unroll
                for (int j = 0; j < QPT; ++j) anyq |= cs[j] == QUEUED;
                if (full && !anyq) {
#pragma unroll
                    for (int c = 0; c < QPT / 4; ++c) {
                        reinterpret_cast<uchar4 *>(qd.codes + q0)[c] =
                            make_uchar4(cs[4 * c], cs[4 * c + 1], cs[4 * c + 2], cs[4 * c + 3]);
                        if (qd.visited) reinterpret_cast<uint4 *>(qd.visited + q0)[c] = make_uint4(0, 0, 0, 0);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < QPT; ++j)
                        if (q0 + j < count && cs[j] != QUEUED) {
                            qd.codes[q0 + j] = cs[j];
                            if (qd.visited) qd.visited[q0 + j] = 0;
                        }
                }
            }
        }
    }
    if constexpr (TBFS && !DBL_EXP_NOBFS) {
        // (the pivot prune is left out here: these BFS expand <= 3 vertices
        // on R-MAT, and its bitmap test adds a dependent load before each
        // record read -- measured 24.2 vs 23.1 us per 1M batch on cfg2)
        __shared__ uint32_t wq[LEAN_THREADS / 32][TB_Q];
        auto answer = [&](uint32_t t) {   // one warp per queued query, neighbours in parallel
            const uint32_t i = dq.i[t];
            uint32_t vc = 0;
            const int r = warp_query_bfs<WDL, WBL>(rec, adj, dq.u[t], dq.v[t], dq.dlo[t], dq.bli[t], dq.blo[t],
                                                   prune_dl, prune_bl, Pivot{}, wq[wid], &vc);
            if (lane == 0) {
                if (r == 2) {
                    const uint32_t pp = atomicAdd(&counters[CNT_PENDING], 1u);
                    DBL_DCHECK(pp < count && i < count);
                    pending[pp] = i;
                } else {
                    DBL_DCHECK(i < count);
                    qd.codes[i] = r ? DBL_BFS_POSITIVE : DBL_BFS_NEGATIVE;
                    if (qd.visited) qd.visited[i] = vc;
                }
            }
            __syncwarp();
        };
        // after the label checks every warp of the CTA takes queued queries,
        // so the CTA pays about one BFS chain however they fell on its warps
        __syncthreads();
        const uint32_t nq = min(dq.n, DQ_CAP);
        const int nwb = blockDim.x >> 5;
        for (uint32_t t = wid; t < nq; t += nwb) answer(t);
    }
    // the last CTA out closes the batch, or tail-launches the warp BFS for the
    // queries the thread BFS could not finish
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&counters[CNT_DONE], 1u) == gridDim.x - 1) {
            __threadfence();
            if (*(volatile uint32_t *)&counters[CNT_PENDING] == 0) {
                close_batch(counters, qd.hres);
            } else {
                counters[CNT_DONE] = 0;
                bfs_warp_kernel<WDL, WBL><<<ha.wgrid, FUSED_THREADS, ha.wsmem, cudaStreamTailLaunch>>>(
                    rec, n, adj, qd, pending, ha.wovf, counters, ha);
            }
        }
    }
}

template <int WDL, int WBL>
__global__ void __launch_bounds__(FUSED_THREADS, DBL_QMINB)
bfs_warp_kernel(const uint64_t *__restrict__ rec, uint32_t n, Adj adj, const QueryDesc qd,
                uint32_t *__restrict__ pending, uint32_t *__restrict__ wovf, uint32_t *__restrict__ counters,
                const HardArgs ha) {
    constexpr int H = WDL + WBL, RW = 2 * H, RS = (int)rec_stride(H), WD = WarpBfs<WDL, WBL>::WD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpBfs<WDL, WBL> &B = reinterpret_cast<WarpBfs<WDL, WBL> *>(smem_raw)[wid];
    const uint32_t flags = qd.flags;
    const bool use_dl = flags & DBL_F_USE_DL, use_bl = flags & DBL_F_USE_BL;
    const bool prune_dl = use_dl && (flags & DBL_F_PRUNE_DL), prune_bl = use_bl && (flags & DBL_F_PRUNE_BL);
    const uint32_t npend = *(volatile uint32_t *)&counters[CNT_PENDING];
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    // equal shares: groups of g <= 32 queries, about one group per warp
    uint32_t g = (npend + nw - 1) / nw;
    g = g < 1 ? 1 : (g > 32 ? 32 : g);
    const uint32_t ngroups = (npend + g - 1) / g;
    for (uint32_t gi = gw; gi < ngroups; gi += nw) {
        const uint32_t p0 = gi * g, nb = min(g, npend - p0);
        if (lane < (int)nb) {
            const uint32_t qi = pending[p0 + lane];
            const uint32_t u = __ldg(qd.u + qi), v = __ldg(qd.v + qi);
            uint64_t ru[RW], rv[RW];
            load_record<RW, RS>(rec + (size_t)u * RS, ru);
            load_record<RW, RS>(rec + (size_t)v * RS, rv);
            B.qidx[lane] = qi;
            B.qu[lane] = u;
            B.qv[lane] = v;
#pragma unroll
            for (int q = 0; q < WDL; ++q) B.qdlo[lane * WD + q] = ru[H + q];
#pragma unroll
            for (int q = 0; q < WBL; ++q) {
                B.qbli[lane * WBL + q] = rv[WDL + q];
                B.qblo[lane * WBL + q] = rv[H + WDL + q];
            }
        }
        if (lane == 0) B.nq = nb;
        __syncwarp();
        warp_bfs_batch<WDL, WBL>(B, rec, adj, prune_dl, prune_bl, qd.pv, qd.codes, qd.visited, wovf, counters, CNT_WOVF);
    }
    // the last CTA out closes the batch, or moves the overflowed queries to
    // the head of the pending list and tail-launches the group/dense kernels
    __syncthreads();
    __shared__ uint32_t last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&counters[CNT_DONE], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const uint32_t nov = *(volatile uint32_t *)&counters[CNT_WOVF];
    if (nov == 0) {
        if (threadIdx.x == 0) close_batch(counters, qd.hres);
        return;
    }
    for (uint32_t i = threadIdx.x; i < nov; i += blockDim.x) pending[i] = wovf[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        counters[CNT_PENDING] = nov;
        __threadfence();
        bfs_kernel<false><<<ha.grid, BFS_THREADS, ha.smem, cudaStreamTailLaunch>>>(
            rec, ha.wdl, ha.wbl, n, adj, qd, pending, counters, ha.ovf, nullptr);
        if (ha.ws)
            bfs_kernel<true><<<ha.dctas, BFS_THREADS, ha.dsmem, cudaStreamTailLaunch>>>(
                rec, ha.wdl, ha.wbl, n, adj, qd, pending, counters, ha.ovf, ha.ws);
        finish_batch_kernel<<<1, 32, 0, cudaStreamTailLaunch>>>(counters, qd.hres);
    }
}

typedef void (*lean_fn)(const uint64_t *, uint32_t, const Adj, const QueryDesc, uint32_t *, uint32_t *,
                        const HardArgs);
typedef void (*bfsw_fn)(const uint64_t *, uint32_t, Adj, const QueryDesc, uint32_t *, uint32_t *, uint32_t *,
                        const HardArgs);

static bool pick_lean(uint32_t wdl, uint32_t wbl, bool qpt4, lean_fn &l, bfsw_fn &b, size_t &smem) {
#define DBL_QL(A, B) if (wdl == A && wbl == B) { l = qpt4 ? label_lean_kernel<A, B, DBL_QPT_HOST> : label_lean_kernel<A, B, 1>; \
        b = bfs_warp_kernel<A, B>; \
        smem = sizeof(WarpBfs<A, B>) * (FUSED_THREADS / 32); return true; }
    DBL_QL(0, 1) DBL_QL(1, 1) DBL_QL(2, 1) DBL_QL(4, 1) DBL_QL(0, 2) DBL_QL(1, 2) DBL_QL(2, 2)
#undef DBL_QL
    return false;
}

typedef void (*quad_fn)(const uint64_t *, uint32_t, Adj, const QueryDesc, uint32_t *, uint32_t *, const HardArgs);

static bool pick_quad(uint32_t wdl, uint32_t wbl, quad_fn &f, size_t &smem) {
#define DBL_QQ(A, B) if (wdl == A && wbl == B) { f = query_quad_kernel<A, B>; smem = sizeof(WarpBfs<A, B>) * (FUSED_THREADS / 32); return true; }
    DBL_QQ(2, 1) DBL_QQ(4, 1) DBL_QQ(1, 2) DBL_QQ(2, 2)
#undef DBL_QQ
    return false;
}

// Launch geometry of the hard path (64-query groups, then dense groups).
struct HardPath {
    int grid = 0, dctas = 0;
    size_t smem = 0, dsmem = 0;
    char *ws = nullptr;
};

static size_t dense_slab(const dbl_index *idx) { return (size_t)idx->n * 32; }

// The dense kernel's workspace (one n x 32-byte slab per CTA) is allocated
// the first time a batch needs it, never up front: at n = 2^30 one slab is
// 32 GB.  A batch that lists dense groups while the workspace is absent
// closes with them unanswered (result words: overflow > 0, dense ticket 0);
// the host then allocates the workspace and re-runs the batch
// (query_needs_dense).  Up to 8 CTAs within min(4 GB, free / 4).
dbl_status ensure_dense(const dbl_index *idx, dbl_graph *g) {
    const size_t slab = dense_slab(idx);
    if (g->q_dense.bytes >= slab + 16) return DBL_OK;
    size_t free_b = 0, total_b = 0;
    DBL_CUDA(cudaMemGetInfo(&free_b, &total_b));
    size_t budget = free_b / 4;
    if (budget > ((size_t)4 << 30)) budget = (size_t)4 << 30;
    size_t ctas = budget / slab;
    if (ctas < 1) ctas = 1;
    if (ctas > 8) ctas = 8;
    dbl_status s = g->q_dense.ensure(slab * ctas + 16);
    if (s && ctas > 1) s = g->q_dense.ensure(slab + 16);
    if (s) set_error("query: the dense BFS workspace (" + std::to_string(slab >> 20) + " MB per CTA) does not fit");
    return s;
}

bool query_needs_dense(const uint32_t *res) { return res[CNT_OVERFLOW] != 0 && res[CNT_DTICKET] == 0; }

static dbl_status hard_path_config(const dbl_index *idx, dbl_graph *g, HardPath &hp) {
    hp.smem = bfs_smem(idx->wdl, idx->wbl, false);
    hp.dsmem = bfs_smem(idx->wdl, idx->wbl, true);
    int bps = 1, dbps = 1;
    dbl_status s;
    if ((s = kernel_occupancy((const void *)bfs_kernel<false>, BFS_THREADS, hp.smem, &bps)) ||
        (s = kernel_occupancy((const void *)bfs_kernel<true>, BFS_THREADS, hp.dsmem, &dbps)))
        return s;
    hp.grid = g->sm_count * bps;
    const size_t slab = dense_slab(idx);
    if (g->q_dense.p && g->q_dense.bytes >= slab + 16) {
        hp.ws = g->q_dense.as<char>();
        size_t c = (g->q_dense.bytes - 16) / slab;
        hp.dctas = (int)(c > 8 ? 8 : c);
    }
    return DBL_OK;
}

// One batch = one launch on the fast path: the gather kernel (K6 + K7)
// takes its arguments by value and leaves the counters zeroed; the warp,
// 64-query group and dense kernels are tail-launched from the device only
// when some query outgrew the previous stage (never on cfg2), so the host
// submits one kernel and no memset, copy or graph per batch.
dbl_status run_query(const dbl_index *idx, dbl_graph *g, const uint32_t *u, const uint32_t *v,
                     uint64_t count, uint32_t flags, uint8_t *codes, uint32_t *visited, bool host_result,
                     bool host_inputs) {
    if (count >= 0xffffffffull) { set_error("query batch too large"); return DBL_E_ARG; }
    if (idx->wdl > MAXW || idx->wbl > MAXW) {
        set_error("label width too large for the query kernels");
        return DBL_E_CONFIG;
    }
    dbl_status s;
    // pending list capacity: grows with the largest batch seen
    uint64_t cap = g->q_pending_cap;
    if (count > cap) cap = count < 1024 ? 1024 : count;
    // pending list [0, cap), dense-group overflow list [cap + 16, 2 cap + 16),
    // warp-batch overflow list [2 cap + 32, 3 cap + 32)
    if ((s = g->q_pending.ensure(cap * 12 + 256))) return s;
    g->q_pending_cap = cap;
    if (!g->q_counters.p) {
        if ((s = g->q_counters.ensure(CNT_ALL * 4))) return s;
        DBL_CUDA(cudaMemsetAsync(g->q_counters.p, 0, CNT_ALL * 4, g->stream));
    }
    if ((s = g->q_host_res.ensure(CNT_WORDS * 4))) return s;
    QueryDesc qd{u, v, codes, visited, (uint32_t)count, flags, 0, 0, Pivot{},
                 host_result ? reinterpret_cast<uint32_t *>(g->q_host_res.p) : nullptr, nullptr};
    if (idx->has_scc && !DBL_NO_PIVOT_PRUNE) {
        qd.pv.dmask = idx->dmask.as<uint32_t>();
        qd.pv.scc = idx->sccmask.as<unsigned long long>();
        qd.pv.n = idx->dmask_n;
    }
    uint32_t *pending = g->q_pending.as<uint32_t>();
    uint32_t *counters = g->q_counters.as<uint32_t>();
    uint32_t *ovf = pending + g->q_pending_cap + 16;
    const uint64_t *rec = idx->rec.as<uint64_t>();
    const Adj adj = graph_fwd(g);
    HardPath hp;
    if ((s = hard_path_config(idx, g, hp))) return s;
    g->q_last = {idx, u, v, codes, visited, count, flags};
    // the digest is used whenever it is current; a stale one (labels changed
    // since) is recomputed only for a batch large enough to repay the
    // n-record pass, small batches read the records directly
    if (DBL_DIGEST && idx->digest_version != idx->version && count >= DBL_DIGEST_REFRESH_MIN &&
        (s = digest_refresh(idx, g)))
        return s;
    if (DBL_DIGEST && idx->digest_version == idx->version) qd.dig = idx->digest.as<uint32_t>();
    lean_fn lean = nullptr;
    bfsw_fn bfsw = nullptr;
    size_t wsmem = 0;
    // k <= 64: lean gather + per-lane deferred BFS.  Wider labels (cfg5,
    // k = 256) take the lean kernel too when the digest is current (it
    // decides ~97% of the pairs, so few records are gathered: cfg5 64M batch
    // 2.65 ms vs 3.91 ms in the quad kernel with the digest, 4.51 ms
    // without), else the lane-quad gather with the warp BFS (measured on
    // cfg5 without the digest: 4.6 vs 3.7 G q/s for the lean gather)
    // pairs in pinned host memory (zero-copy): 4 pairs per thread per step
    // when the buffers allow the vector loads and stores
    const bool qpt4 = (host_inputs || DBL_QPT_DEV) && ((((uintptr_t)u) | ((uintptr_t)v)) & 15) == 0 && (((uintptr_t)codes) & 3) == 0 &&
                      (!visited || (((uintptr_t)visited) & 15) == 0);
    if (count && (DBL_TBFS_ALL || DBL_LEAN_WIDE || idx->wdl <= 1 || qd.dig) &&
        pick_lean(idx->wdl, idx->wbl, qpt4, lean, bfsw, wsmem)) {
        int lbps = 1, wbps = 1;
        if ((s = kernel_occupancy((const void *)lean, LEAN_THREADS, 0, &lbps)) ||
            (s = kernel_occupancy((const void *)bfsw, FUSED_THREADS, wsmem, &wbps)))
            return s;
        uint32_t *wovf = pending + 2 * g->q_pending_cap + 32;
        const HardArgs ha{hp.grid, hp.dctas, (uint32_t)hp.smem, (uint32_t)hp.dsmem, idx->wdl, idx->wbl, ovf,
                          hp.ws, g->sm_count * wbps, (uint32_t)wsmem, wovf};
        const uint64_t per = qpt4 ? DBL_QPT_HOST * LEAN_THREADS : LEAN_THREADS;   // queries per CTA per step
        uint32_t lgrid = (uint32_t)((count + per - 1) / per);
        if (lgrid > (uint32_t)(g->sm_count * lbps * DBL_LEAN_WAVES)) lgrid = (uint32_t)(g->sm_count * lbps * DBL_LEAN_WAVES);
        if (g->instrument) DBL_CUDA(cudaEventRecord(g->ev[2], g->stream));
        lean<<<lgrid, LEAN_THREADS, 0, g->stream>>>(rec, idx->n, adj, qd, pending, counters, ha);
        DBL_CHECK_LAUNCH("label_lean_kernel");
        if (g->instrument) DBL_CUDA(cudaEventRecord(g->ev[3], g->stream));
        g->q_timed_bfs = false;
        return DBL_OK;
    }
    quad_fn quad = nullptr;
    size_t fsmem = 0;
    if (count && pick_quad(idx->wdl, idx->wbl, quad, fsmem)) {
        int fbps = 1;
        if ((s = kernel_occupancy((const void *)quad, FUSED_THREADS, fsmem, &fbps))) return s;
        const HardArgs ha{hp.grid, hp.dctas, (uint32_t)hp.smem, (uint32_t)hp.dsmem, idx->wdl, idx->wbl, ovf, hp.ws};
        if (g->instrument) DBL_CUDA(cudaEventRecord(g->ev[2], g->stream));
        quad<<<g->sm_count * fbps, FUSED_THREADS, fsmem, g->stream>>>(rec, idx->n, adj, qd, pending, counters, ha);
        DBL_CHECK_LAUNCH("query_quad_kernel");
        if (g->instrument) DBL_CUDA(cudaEventRecord(g->ev[3], g->stream));
        g->q_timed_bfs = false;
        return DBL_OK;
    }
    // generic widths (k > 256 or k' > 128): label kernel, then the group and
    // dense kernels, then the counter close
    if (g->instrument) DBL_CUDA(cudaEventRecord(g->ev[2], g->stream));
    if (count) {
        int blocks = (int)((count + 255) / 256);
        if (blocks > g->sm_count * 16) blocks = g->sm_count * 16;
        label_check_generic<<<blocks, 256, 0, g->stream>>>(rec, idx->n, idx->wdl, idx->wbl, u, v, count, flags,
                                                           codes, visited, pending, counters);
        DBL_CHECK_LAUNCH("label_check_generic");
    }
    if (g->instrument) DBL_CUDA(cudaEventRecord(g->ev[3], g->stream));
    if (count) {
        bfs_kernel<false><<<hp.grid, BFS_THREADS, hp.smem, g->stream>>>(rec, idx->wdl, idx->wbl, idx->n, adj, qd,
                                                                        pending, counters, ovf, nullptr);
        DBL_CHECK_LAUNCH("bfs_kernel");
        if (hp.ws) {
            bfs_kernel<true><<<hp.dctas, BFS_THREADS, hp.dsmem, g->stream>>>(rec, idx->wdl, idx->wbl, idx->n, adj,
                                                                             qd, pending, counters, ovf, hp.ws);
            DBL_CHECK_LAUNCH("bfs_kernel_dense");
        }
    }
    finish_batch_kernel<<<1, 32, 0, g->stream>>>(counters, qd.hres);
    DBL_CHECK_LAUNCH("finish_batch_kernel");
    if (g->instrument) DBL_CUDA(cudaEventRecord(g->ev[4], g->stream));
    g->q_timed_bfs = true;
    return DBL_OK;
}

// Copy result words [ERR, DTICKET] of the last batch (range-error flag,
// group ticket, dense-group count, dense ticket) to dst[0..3] (device,
// stream-ordered): the chunked host pipeline keeps one set per chunk.
dbl_status query_err_to(dbl_graph *g, uint32_t *dst) {
    DBL_CUDA(cudaMemcpyAsync(dst, g->q_counters.as<uint32_t>() + CNT_RES + CNT_ERR, 4 * 4, cudaMemcpyDeviceToDevice,
                             g->stream));
    return DBL_OK;
}

bool chunk_needs_dense(const uint32_t *w4) { return w4[CNT_OVERFLOW - CNT_ERR] != 0 && w4[CNT_DTICKET - CNT_ERR] == 0; }

// Event times of the last batch: the gather kernel's span (incl. any
// tail-launched hard path) as "label", the separate BFS kernels as "bfs".
void query_timings(dbl_graph *g) {
    g->t_label = g->t_bfs = 0;
    if (!g->instrument) return;   // per-launch events only on instrumented graphs
    cudaEventElapsedTime(&g->t_label, g->ev[2], g->ev[3]);
    g->t_bfs = 0;
    if (g->q_timed_bfs) cudaEventElapsedTime(&g->t_bfs, g->ev[3], g->ev[4]);
}

// Wait for the batch; *err_out = range-error flag, *dense_out = it left
// groups for a dense workspace that was not allocated yet.  The closing CTA
// wrote the result words into the pinned q_host_res, so the stream sync is
// the batch's only host step (timings are read lazily by dbl_last_timings).
dbl_status query_finish(dbl_graph *g, uint32_t *err_out, bool *dense_out) {
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    const volatile uint32_t *r = reinterpret_cast<const volatile uint32_t *>(g->q_host_res.p);
    uint32_t w[CNT_WORDS];
    for (int i = 0; i < CNT_WORDS; ++i) w[i] = r[i];
    *err_out = w[CNT_ERR];
    *dense_out = query_needs_dense(w);
    return DBL_OK;
}

// dbl_sync: wait for the stream; if the last batch (an async one) left dense
// groups, allocate the workspace and re-run it with the same arguments.
dbl_status query_sync(dbl_graph *g) {
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    if (!g->q_counters.p || !g->q_last.idx) return DBL_OK;
    uint32_t w[CNT_WORDS];
    DBL_CUDA(cudaMemcpy(w, g->q_counters.as<uint32_t>() + CNT_RES, sizeof(w), cudaMemcpyDeviceToHost));
    if (!query_needs_dense(w)) return DBL_OK;
    const QueryArgs a = g->q_last;
    dbl_status s;
    if ((s = ensure_dense(a.idx, g))) return s;
    if ((s = run_query(a.idx, g, a.u, a.v, a.count, a.flags, a.codes, a.visited))) return s;
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    return DBL_OK;
}

// ------------------------------------------------- per-call service (K6s) --
//
// A single query() or insert_edge() call used to pay a kernel launch and a
// stream sync (10.1 us on this box for an empty kernel, tools/ubench_api.cu)
// on top of a few microseconds of work.  The service keeps one CTA resident
// that polls a mailbox in pinned host memory (round trip 2.4 us, same tool):
//   * a query (u, v, flags): warp 0 applies K6's rules (digest, then both
//     records, rules 1-4 in order, queries.py:96-114) and, if they leave it
//     open, the bounded warp BFS (queries.py:116-142); a query that outgrows
//     the BFS, or needs one after the service inserted edges (they sit in the
//     pending log, which the BFS does not read), is handed back to the batch
//     path;
//   * an insert (u, v): the whole CTA runs K9 (insert_one.cuh,
//     updates.py:112-137) against the pending log; a cone beyond K9's tables
//     is handed back to the batch fixpoint, as from the K9 launch.
// The CTA exits after SERVE_IDLE_NS without a request; every other entry
// point of the library stops it first (serve_quiesce), so it never runs
// beside another label or adjacency write or a cooperative launch.  Records
// and digests are read L2-coherently (.cg): the service writes them itself.
//
// Request and answer are one 16-byte word each, written and read with single
// vector accesses (one PCIe transaction each way); the sequence number is
// the last word the host writes (x86 keeps store order), so a request read
// with the new sequence number also holds its own fields.
struct alignas(64) ServeBox {
    uint32_t u, v, opflags, seq, pad0[12];              // host -> device: op << 16 | (flags or pending count)
    uint32_t code, visited, status, rseq, pad1[12];     // device -> host (own line)
    OneOut ins;                                         // insert result (written before the answer word)
    uint32_t alive, pad2[3];
};
enum { SERVE_QUERY = 1, SERVE_STOP = 2, SERVE_INSERT = 3 };
enum { SERVE_OK = 0, SERVE_FALLBACK = 1 };
#ifndef DBL_SERVE
#define DBL_SERVE 1                 // 0: single calls take the launch + sync path
#endif
constexpr uint64_t SERVE_IDLE_NS = 2000000;   // the CTA exits after 2 ms without a request

__device__ __forceinline__ uint64_t serve_clock() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int RW, int RS>
__device__ __forceinline__ void load_record_cg(const uint64_t *p, uint64_t (&r)[RW]) {
    constexpr int V4 = RS % 4 == 0 ? RW / 4 * 4 : 0;
#pragma unroll
    for (int k = 0; k < V4; k += 4)
        asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(r[k]), "=l"(r[k + 1]), "=l"(r[k + 2]), "=l"(r[k + 3]) : "l"(p + k));
#pragma unroll
    for (int k = V4; k < RW; k += 2)
        asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(r[k]), "=l"(r[k + 1]) : "l"(p + k));
}

struct ServeArgs {
    uint64_t *rec;
    const uint32_t *dig;    // current digest or nullptr (inserts keep it current)
    uint32_t n;
    Adj fwd, rev;
    uint64_t *pend;         // single-edge log (device)
    ServeBox *box;          // device address of the pinned mailbox
    uint32_t start_seq;
};

template <int WDL, int WBL>
__global__ void __launch_bounds__(ONE_THREADS, 1) serve_kernel(const ServeArgs A) {
    constexpr int H = WDL + WBL, RW = 2 * H, RS = (int)rec_stride(H), WD = WDL > 0 ? WDL : 1;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t wq[TB_Q];
    __shared__ uint64_t sdlo[WD], sbli[WBL], sblo[WBL];
    __shared__ uint32_t req[4];
    ServeBox *box = A.box;
    const int tid = threadIdx.x, lane = tid & 31;
    uint32_t last = A.start_seq;
    bool dirty = false;   // the service inserted edges: its BFS would miss the pending ones
    uint64_t t_idle = serve_clock();
    for (;;) {
        if (tid == 0) {
            uint32_t u, v, opflags, seq;
            for (;;) {
                asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(u), "=r"(v), "=r"(opflags), "=r"(seq) : "l"(box) : "memory");
                if (seq != last || serve_clock() - t_idle > SERVE_IDLE_NS) break;
            }
            req[0] = u; req[1] = v; req[2] = seq == last ? (SERVE_STOP << 16) : opflags; req[3] = seq;
        }
        __syncthreads();
        const uint32_t u = req[0], v = req[1], opflags = req[2], seq = req[3], op = opflags >> 16;
        __syncthreads();
        if (op == SERVE_INSERT) {
            insert_one_body(A.rec, RS, H, WDL, A.n, u, v, A.fwd, A.rev, A.pend, opflags & 0xffffu, PEND_CAP,
                            &box->ins, const_cast<uint32_t *>(A.dig), reinterpret_cast<OneShared *>(smem));
            dirty = true;
            __syncthreads();
            if (tid == 0) {
                __threadfence_system();   // the OneOut lands before the answer word
                asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1, %2, %3, %4};"
                             ::"l"(&box->code), "r"(0u), "r"(0u), "r"((uint32_t)SERVE_OK), "r"(seq) : "memory");
            }
        } else if (op == SERVE_QUERY) {
            if (tid < 32) {
                const uint32_t flags = opflags & 0xffffu;
                const bool use_dl = flags & DBL_F_USE_DL, use_bl = flags & DBL_F_USE_BL;
                const bool thm1 = use_dl && (flags & DBL_F_THM1), thm2 = use_dl && (flags & DBL_F_THM2);
                const bool prune_dl = use_dl && (flags & DBL_F_PRUNE_DL), prune_bl = use_bl && (flags & DBL_F_PRUNE_BL);
                uint32_t code = UNRESOLVED, vc = 0, status = SERVE_OK;
                if (u >= A.n || v >= A.n) {
                    status = SERVE_FALLBACK;   // (the host checks the range first)
                } else if (u == v) {
                    code = DBL_REFLEXIVE;
                } else {
                    if (A.dig) code = digest_decide(__ldcg(A.dig + u), __ldcg(A.dig + v), use_dl, use_bl);
                    if (code == UNRESOLVED) {
                        uint64_t a[RW], b[RW];
                        load_record_cg<RW, RS>(A.rec + (size_t)u * RS, a);
                        load_record_cg<RW, RS>(A.rec + (size_t)v * RS, b);
                        uint64_t r1 = 0, r2 = 0, r3 = 0, r4 = 0;
#pragma unroll
                        for (int k = 0; k < WDL; ++k) {
                            r1 |= a[H + k] & b[k];
                            r3 |= b[H + k] & a[k];
                            r4 |= (a[H + k] & a[k]) | (b[H + k] & b[k]);
                        }
#pragma unroll
                        for (int k = 0; k < WBL; ++k)
                            r2 |= (a[WDL + k] & ~b[WDL + k]) | (b[H + WDL + k] & ~a[H + WDL + k]);
                        if (use_dl && r1) code = DBL_DL_POSITIVE;
                        else if (use_bl && r2) code = DBL_BL_NEGATIVE;
                        else if (thm1 && r3) code = DBL_THM1_NEGATIVE;
                        else if (thm2 && r4) code = DBL_THM2_NEGATIVE;
                        if (code == UNRESOLVED && dirty) {
                            status = SERVE_FALLBACK;
                        } else if (code == UNRESOLVED) {
                            if (lane == 0) {
#pragma unroll
                                for (int k = 0; k < WDL; ++k) sdlo[k] = a[H + k];
#pragma unroll
                                for (int k = 0; k < WBL; ++k) {
                                    sbli[k] = b[WDL + k];
                                    sblo[k] = b[H + WDL + k];
                                }
                            }
                            __syncwarp();
                            const int r = warp_query_bfs<WDL, WBL>(A.rec, A.fwd, u, v, sdlo, sbli, sblo, prune_dl,
                                                                   prune_bl, Pivot{}, wq, &vc);
                            if (r == 2) status = SERVE_FALLBACK;
                            else code = r ? DBL_BFS_POSITIVE : DBL_BFS_NEGATIVE;
                            __syncwarp();
                        }
                    }
                }
                if (lane == 0)
                    asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1, %2, %3, %4};"
                                 ::"l"(&box->code), "r"(code), "r"(vc), "r"(status), "r"(seq) : "memory");
            }
        } else {
            break;   // stop, idle, or an unknown request
        }
        last = seq;
        t_idle = serve_clock();
    }
    if (tid == 0) st_release_sys(&box->alive, 0u);
}

typedef void (*serve_fn)(const ServeArgs);

static serve_fn pick_serve(uint32_t wdl, uint32_t wbl) {
#define DBL_SV(A, B) if (wdl == A && wbl == B) return serve_kernel<A, B>;
    DBL_SV(0, 1) DBL_SV(1, 1) DBL_SV(2, 1) DBL_SV(4, 1) DBL_SV(0, 2) DBL_SV(1, 2) DBL_SV(2, 2)
#undef DBL_SV
    return nullptr;
}

// One service at a time per process (it holds one SM); the mutex also
// serialises concurrent single calls, which share the mailbox.
static std::mutex g_srv_mu;
static dbl_graph *g_srv = nullptr;
static std::atomic<int> g_srv_on{0};
// A service launched for a request that exits without answering it means
// kernel launches block until the kernel ends (a profiler or sanitizer
// serialising launches, CUDA_LAUNCH_BLOCKING): single calls then take the
// launch path for the rest of the process.
static bool g_srv_off = false;

static void post_stop(dbl_graph *g) {
    volatile ServeBox *vb = reinterpret_cast<volatile ServeBox *>(g->sbox.p);
    vb->opflags = SERVE_STOP << 16;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    vb->seq = ++g->s_seq;
}

static void serve_stop_locked() {
    dbl_graph *g = g_srv;
    if (!g) return;
    g_srv = nullptr;
    g_srv_on.store(0, std::memory_order_release);
    if (!g->s_running) return;
    post_stop(g);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaSetDevice(g->device);
    cudaStreamSynchronize(g->sstream);
    cudaSetDevice(dev);
    g->s_running = false;
}

void serve_quiesce() {
    if (g_srv_on.load(std::memory_order_acquire) == 0) return;
    std::lock_guard<std::mutex> lk(g_srv_mu);
    serve_stop_locked();
}

static std::atomic<int> g_srv_block{0};
ServeBlock::ServeBlock() {
    g_srv_block.fetch_add(1, std::memory_order_acq_rel);
    serve_quiesce();
}
ServeBlock::~ServeBlock() { g_srv_block.fetch_sub(1, std::memory_order_acq_rel); }

// Release the graph's service resources (dbl_graph_free, after serve_quiesce).
void serve_release(dbl_graph *g) {
    if (g->sstream) {
        cudaStreamSynchronize(g->sstream);
        cudaStreamDestroy(g->sstream);
        g->sstream = nullptr;
    }
    g->sbox.release();
}

static dbl_status serve_start_locked(const dbl_index *idx, dbl_graph *g, serve_fn fn) {
    if (g_srv != g) serve_stop_locked();
    DBL_CUDA(cudaSetDevice(g->device));
    dbl_status s;
    if (g->s_running) {   // an exited (idle) or outdated service of this graph
        post_stop(g);
        DBL_CUDA(cudaStreamSynchronize(g->sstream));
        g->s_running = false;
    }
    // the query BFS reads the adjacency: fold the single-edge log in first,
    // and let the engine stream's queued work (builds, inserts) finish
    set_stream(g->stream);
    if ((s = graph_flush_pending(g))) return s;
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    const size_t smem = 2 * sizeof(OneShared);
    int bps = 0;
    if ((s = kernel_occupancy((const void *)fn, ONE_THREADS, smem, &bps))) return s;
    if ((s = g->sbox.ensure(sizeof(ServeBox) + 64)) || (s = g->pend.ensure(PEND_CAP * 8 + 64))) return s;
    if (!g->sstream) DBL_CUDA(cudaStreamCreateWithFlags(&g->sstream, cudaStreamNonBlocking));
    ServeBox *hb = reinterpret_cast<ServeBox *>(g->sbox.p);
    ServeBox *db = nullptr;
    DBL_CUDA(cudaHostGetDevicePointer((void **)&db, hb, 0));
    volatile ServeBox *vb = hb;
    vb->rseq = g->s_seq;
    vb->seq = g->s_seq;
    vb->alive = 1;
    static_assert(offsetof(ServeBox, code) % 16 == 0 && offsetof(ServeBox, rseq) == offsetof(ServeBox, code) + 12,
                  "the answer is one 16-byte word");
    std::atomic_thread_fence(std::memory_order_seq_cst);
    ServeArgs A{const_cast<uint64_t *>(idx->rec.as<uint64_t>()),
                DBL_DIGEST && idx->digest_version == idx->version ? idx->digest.as<uint32_t>() : nullptr,
                idx->n, graph_fwd(g), graph_rev(g), g->pend.as<uint64_t>(), db, g->s_seq};
    g->s_dig = A.dig != nullptr;
    fn<<<1, ONE_THREADS, smem, g->sstream>>>(A);
    DBL_CHECK_LAUNCH("serve_kernel");
    g->s_running = true;
    g->s_idx = idx;
    g->s_ver = idx->version;
    g_srv = g;
    g_srv_on.store(1, std::memory_order_release);
    return DBL_OK;
}

// Post one request and wait for its answer word (code, visited, status).
// op = SERVE_INSERT sends the pending-log length (read after any restart,
// which folds the log in).  *served = false: no service kernel for these
// label widths.
static dbl_status serve_call(const dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v, uint32_t op,
                             uint32_t flags, uint32_t ans[3], bool *served) {
    *served = false;
    const serve_fn fn = DBL_SERVE ? pick_serve(idx->wdl, idx->wbl) : nullptr;
    // another thread is inside a library call: take the launch path (a
    // service started now would be stopped by it anyway)
    if (!fn || g_srv_off || g_srv_block.load(std::memory_order_acquire) > 0) return DBL_OK;
    dbl_status s;
    for (int attempt = 0; attempt < 3; ++attempt) {
        bool fresh = false;
        if (g_srv != g || !g->s_running || g->s_idx != idx || g->s_ver != idx->version ||
            (op == SERVE_INSERT && g->n_pend >= PEND_CAP) ||
            reinterpret_cast<volatile ServeBox *>(g->sbox.p)->alive == 0) {
            if ((s = serve_start_locked(idx, g, fn))) return s;
            fresh = true;
        }
        volatile ServeBox *vb = reinterpret_cast<volatile ServeBox *>(g->sbox.p);
        vb->u = u;
        vb->v = v;
        vb->opflags = (op << 16) | ((op == SERVE_INSERT ? g->n_pend : flags) & 0xffffu);
        std::atomic_signal_fence(std::memory_order_seq_cst);   // the sequence number is stored last
        const uint32_t seq = ++g->s_seq;
        vb->seq = seq;
        const auto t0 = std::chrono::steady_clock::now();
        for (uint32_t it = 0;; ++it) {
            alignas(16) uint32_t w[4];   // one 16-byte load: the answer and its sequence number together
            _mm_store_si128(reinterpret_cast<__m128i *>(w),
                            _mm_load_si128(reinterpret_cast<const __m128i *>(const_cast<uint32_t *>(&vb->code))));
            if (w[3] == seq) {
                ans[0] = w[0];
                ans[1] = w[1];
                ans[2] = w[2];
                std::atomic_thread_fence(std::memory_order_acquire);
                *served = true;
                return DBL_OK;
            }
            if (vb->alive == 0) {   // went idle just before the request: relaunch, post again
                if (vb->rseq == seq) continue;
                g->s_running = false;
                cudaStreamSynchronize(g->sstream);
                if (fresh) {   // a fresh service never saw its first request: launches block
                    g_srv_off = true;
                    serve_stop_locked();
                    return DBL_OK;
                }
                break;
            }
            if ((it & 1023) == 1023 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
                serve_stop_locked();
                set_error("per-call service did not answer within 2 s");
                return DBL_E_CUDA;
            }
        }
    }
    return DBL_OK;   // (not reached in practice) the launch path answers it
}

// Answer one query through the service.  *served = false: the caller answers
// it on the batch path (no service kernel for these widths, or the service
// handed it back).
dbl_status serve_query(const dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v, uint32_t flags, uint8_t *code,
                       uint32_t *visited, bool *served) {
    std::lock_guard<std::mutex> lk(g_srv_mu);
    uint32_t ans[3];
    dbl_status s = serve_call(idx, g, u, v, SERVE_QUERY, flags, ans, served);
    if (s || !*served) return s;
    if (ans[2] != SERVE_OK) {
        *served = false;
        serve_stop_locked();   // the batch path takes it (its BFS stages run on the engine stream)
        return DBL_OK;
    }
    *code = (uint8_t)ans[0];
    if (visited) *visited = ans[1];
    return DBL_OK;
}

dbl_status serve_insert(dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v, dbl_update_stats *st, bool *done,
                        uint32_t *dirs_done, bool *dig_ok, bool *served) {
    std::lock_guard<std::mutex> lk(g_srv_mu);
    *served = false;
    if (idx->wdl + idx->wbl > (uint32_t)MAX_SHARD_WORDS) return DBL_OK;
    uint32_t ans[3];
    dbl_status s = serve_call(idx, g, u, v, SERVE_INSERT, 0, ans, served);
    if (s || !*served) return s;
    OneOut o;
    const volatile OneOut *vo = &reinterpret_cast<volatile ServeBox *>(g->sbox.p)->ins;
    std::memcpy(&o, const_cast<const OneOut *>(vo), sizeof(o));
    // labels may have changed: the version moves; the service wrote the
    // digest bits too iff it holds the digest, and it reads the new labels
    // itself, so it stays valid for the next call
    *dig_ok = g->s_dig;
    ++idx->version;
    if (g->s_dig) idx->digest_version = idx->version;
    g->s_ver = idx->version;
    s = insert_edge_outcome(g, o, st, done, dirs_done);
    if (s || !*done) serve_stop_locked();   // the batch fixpoint finishes it (cooperative launch)
    return s;
}

}  // namespace dbl

using namespace dbl;

// The index's query digest (n u32, host), recomputed first if stale.
extern "C" dbl_status dbl_index_digest(const dbl_index *idx, const dbl_graph *gc, uint32_t *out,
                                       int *was_current) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx || !gc || (!out && idx->n)) { set_error("null argument"); return DBL_E_ARG; }
    if (was_current) *was_current = idx->digest_version == idx->version;
    if (idx->n != gc->n) { set_error("graph and index vertex counts differ"); return DBL_E_MISMATCH; }
    dbl_graph *g = const_cast<dbl_graph *>(gc);
    DBL_CUDA(cudaSetDevice(g->device));
    set_stream(g->stream);
    if (!DBL_DIGEST) { set_error("library built without the query digest"); return DBL_E_CONFIG; }
    dbl_status s = digest_refresh(idx, g);
    if (s) return s;
    if (idx->n)
        DBL_CUDA(cudaMemcpyAsync(out, idx->digest.p, (size_t)idx->n * 4, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    return DBL_OK;
}

// Counters of the last query batch on g: [0] queries handed to the group
// kernels (per-warp BFS table overflow or generic widths), [1] range-error
// flag, [3] groups re-run densely.
extern "C" dbl_status dbl_query_counters(const dbl_graph *g, uint32_t *out8) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!g || !out8) { set_error("null argument"); return DBL_E_ARG; }
    if (!g->q_counters.p) { for (int i = 0; i < 8; ++i) out8[i] = 0; return DBL_OK; }
    DBL_CUDA(cudaSetDevice(g->device));
    DBL_CUDA(cudaMemcpyAsync(out8, g->q_counters.as<uint32_t>() + CNT_RES, 8 * 4, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    return DBL_OK;
}
