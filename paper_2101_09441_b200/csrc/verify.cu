// verify.cu -- on-GPU label verifier (reference verify_labels, updates.py:323-363).
//
// Union-fixpoint check (Eq. (1) of the paper): every in-half must equal the
// vertex's own seed bits OR the in-halves of its predecessors; every out-half
// the seed bits OR the out-halves of its successors.  One warp per vertex
// reduces the neighbours' words with lane-strided loads + a shuffle OR tree.
// Exhaustive mode also rebuilds the labels from the frozen metadata and diffs
// the two record tables, which catches stale bits a cycle sustains through
// the fixpoint (the same blind spot the reference covers with its rebuild).
// Violations are data: (vertex, half, expected words, actual words) rows.
#include "internal.cuh"

namespace dbl {

struct ViolationOut {
    unsigned long long *count;
    uint64_t max_out;
    uint32_t *vertex;
    uint8_t *half;
    uint64_t *expected;   // max_out x H words
    uint64_t *actual;
};

__device__ __forceinline__ void emit_violation(const ViolationOut &o, uint32_t H, uint32_t v, uint32_t h,
                                               const uint64_t *exp, const uint64_t *act) {
    const unsigned long long slot = atomicAdd(o.count, 1ull);
    if (slot >= o.max_out) return;
    o.vertex[slot] = v;
    o.half[slot] = (uint8_t)h;
    for (uint32_t w = 0; w < H; ++w) {
        o.expected[slot * H + w] = exp[w];
        o.actual[slot * H + w] = act[w];
    }
}

__global__ void landmark_pos_kernel(const uint32_t *__restrict__ lm, uint32_t k, uint32_t *__restrict__ pos) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) pos[lm[i]] = i;
}

constexpr int VMAXH = 32;

// warp per (vertex, half)
__global__ void fixpoint_check_kernel(const uint64_t *__restrict__ rec, uint32_t n, uint32_t wdl, uint32_t wbl,
                                      Adj fwd, Adj rev, const uint32_t *__restrict__ lmpos,
                                      const uint8_t *__restrict__ flags, const uint32_t *__restrict__ bucket,
                                      ViolationOut out) {
    const uint32_t H = wdl + wbl, rw = rec_stride(H);
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = warp; t < 2ull * n; t += nwarps) {
        const uint32_t v = (uint32_t)(t >> 1), h = (uint32_t)(t & 1);
        const Adj &sup = h == 0 ? rev : fwd;   // in-half: predecessors; out-half: successors
        uint64_t acc[VMAXH];
        for (uint32_t w = 0; w < H; ++w) acc[w] = 0;
        for (int seg = 0; seg < 2; ++seg) {
            const uint32_t *ptr = seg ? sup.dptr : sup.ptr;
            const uint32_t *col = seg ? sup.dcol : sup.col;
            if (!ptr) continue;
            const uint32_t s = ptr[v], e = ptr[v + 1];
            for (uint32_t i = s + lane; i < e; i += 32) {
                const uint64_t *r = rec + (size_t)col[i] * rw + h * H;
                for (uint32_t w = 0; w < H; ++w) acc[w] |= r[w];
            }
        }
        for (uint32_t w = 0; w < H; ++w) {
            uint64_t x = acc[w];
            for (int o = 16; o > 0; o >>= 1) x |= __shfl_xor_sync(FULL, x, o);
            acc[w] = x;
        }
        if (lane == 0) {
            // own seed bits (labels.py:291-305 seeds)
            const uint32_t lp = lmpos[v];
            if (lp != 0xffffffffu) acc[lp / 64] |= 1ull << (lp % 64);
            const uint8_t f = flags[v];
            if ((f >> h) & 1) acc[wdl + bucket[v] / 64] |= 1ull << (bucket[v] % 64);
            const uint64_t *mine = rec + (size_t)v * rw + h * H;
            bool bad = false;
            for (uint32_t w = 0; w < H; ++w) bad |= acc[w] != mine[w];
            if (bad) {
                uint64_t act[VMAXH];
                for (uint32_t w = 0; w < H; ++w) act[w] = mine[w];
                emit_violation(out, H, v, h, acc, act);
            }
        }
    }
}

// exhaustive mode: diff against a fresh rebuild (expected = b)
__global__ void record_diff_kernel(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b, uint32_t n,
                                   uint32_t H, ViolationOut out) {
    const uint32_t rw = rec_stride(H);
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < 2ull * n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)(t >> 1), h = (uint32_t)(t & 1);
        const uint64_t *x = a + (size_t)v * rw + h * H, *y = b + (size_t)v * rw + h * H;
        bool bad = false;
        for (uint32_t w = 0; w < H; ++w) bad |= x[w] != y[w];
        if (bad) emit_violation(out, H, v, h, y, x);
    }
}

}  // namespace dbl

using namespace dbl;

extern "C" dbl_status dbl_verify(const dbl_index *idx, const dbl_graph *gc, int exhaustive, uint64_t max_out,
                                 uint64_t *out_count, uint32_t *out_vertex, uint8_t *out_half,
                                 uint64_t *out_expected, uint64_t *out_actual) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx || !gc || !out_count) { set_error("null argument"); return DBL_E_ARG; }
    if (idx->n != gc->n) {
        set_error("graph and index vertex counts differ");
        return DBL_E_MISMATCH;
    }
    dbl_graph *g = const_cast<dbl_graph *>(gc);
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    const uint32_t n = idx->n, H = idx->wdl + idx->wbl;
    if (H > (uint32_t)VMAXH) { set_error("label width too large for the verifier"); return DBL_E_CONFIG; }
    DevBuf lmpos, cnt, ov, oh, oe, oa;
    auto cleanup = [&]() { lmpos.release(); cnt.release(); ov.release(); oh.release(); oe.release(); oa.release(); };
    dbl_status s;
    const uint64_t mo = max_out ? max_out : 1;
    if ((s = lmpos.ensure((size_t)n * 4 + 4)) || (s = cnt.ensure(8)) || (s = ov.ensure(mo * 4)) ||
        (s = oh.ensure(mo)) || (s = oe.ensure(mo * H * 8 + 8)) || (s = oa.ensure(mo * H * 8 + 8))) {
        cleanup();
        return s;
    }
    DBL_CUDA(cudaMemsetAsync(lmpos.p, 0xff, (size_t)n * 4, g->stream));
    DBL_CUDA(cudaMemsetAsync(cnt.p, 0, 8, g->stream));
    if (idx->cfg.k) {
        landmark_pos_kernel<<<(idx->cfg.k + 255) / 256, 256, 0, g->stream>>>(idx->landmarks.as<uint32_t>(),
                                                                          idx->cfg.k, lmpos.as<uint32_t>());
        DBL_CHECK_LAUNCH("landmark_pos_kernel");
    }
    ViolationOut o{cnt.as<unsigned long long>(), max_out, ov.as<uint32_t>(), oh.as<uint8_t>(), oe.as<uint64_t>(),
                   oa.as<uint64_t>()};
    if (n) {
        fixpoint_check_kernel<<<g->sm_count * 8, 256, 0, g->stream>>>(
            idx->rec.as<uint64_t>(), n, idx->wdl, idx->wbl, graph_fwd(g), graph_rev(g), lmpos.as<uint32_t>(),
            idx->leaf_flags.as<uint8_t>(), idx->bucket.as<uint32_t>(), o);
        DBL_CHECK_LAUNCH("fixpoint_check_kernel");
    }
    if (exhaustive && n) {
        // fresh rebuild with the frozen metadata into a scratch index
        dbl_index fresh;
        fresh.device = idx->device;
        fresh.n = n;
        fresh.cfg = idx->cfg;
        fresh.wdl = idx->wdl;
        fresh.wbl = idx->wbl;
        fresh.rw = idx->rw;
        fresh.rs = idx->rs;
        fresh.landmarks.p = idx->landmarks.p;
        fresh.leaf_flags.p = idx->leaf_flags.p;
        fresh.bucket.p = idx->bucket.p;
        s = fresh.rec.ensure((size_t)n * idx->rs * 8 + 16);
        if (!s) s = run_build(g, &fresh, nullptr, 0);
        if (!s) {
            record_diff_kernel<<<g->sm_count * 8, 256, 0, g->stream>>>(idx->rec.as<uint64_t>(),
                                                                    fresh.rec.as<uint64_t>(), n, H, o);
            DBL_LAUNCHED();
        }
        fresh.rec.release();
        fresh.landmarks.p = fresh.leaf_flags.p = fresh.bucket.p = nullptr;
        if (s) { cleanup(); return s; }
    }
    unsigned long long hc = 0;
    DBL_CUDA(cudaMemcpyAsync(&hc, cnt.p, 8, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    *out_count = hc;
    const uint64_t k = hc < max_out ? hc : max_out;
    if (k) {
        if (out_vertex) DBL_CUDA(cudaMemcpy(out_vertex, ov.p, k * 4, cudaMemcpyDeviceToHost));
        if (out_half) DBL_CUDA(cudaMemcpy(out_half, oh.p, k, cudaMemcpyDeviceToHost));
        if (out_expected) DBL_CUDA(cudaMemcpy(out_expected, oe.p, k * H * 8, cudaMemcpyDeviceToHost));
        if (out_actual) DBL_CUDA(cudaMemcpy(out_actual, oa.p, k * H * 8, cudaMemcpyDeviceToHost));
    }
    cleanup();
    return DBL_OK;
}
