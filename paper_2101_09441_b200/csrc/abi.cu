// abi.cu -- extern "C" entry points for index build, queries and insertion.
// See include/dbl_b200.h for the contract and the reference function each
// entry point replaces.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace dbl {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
std::atomic<uint64_t> &launch_counter() { return g_launches; }

// ------------------------------------------------------ caching allocator --
// Each cached block remembers the stream that last used it (the calling
// thread's current engine stream, see set_stream); handing it to work on a
// different stream first waits for that stream, so recycled memory is never
// written while an earlier kernel may still read it.
// A block freed right after a device-wide synchronisation (index / graph
// teardown) is "clean": no work can still touch it, so reusing it needs no
// wait at all (a device sync on reuse would sit inside the next build).
struct PoolBlock { void *p; cudaStream_t s; bool clean; };
static std::mutex g_pool_mu;
static std::map<std::pair<int, size_t>, std::vector<PoolBlock>> g_pool;
static thread_local cudaStream_t g_cur_stream = nullptr;
static thread_local bool g_free_clean = false;

void set_stream(cudaStream_t s) { g_cur_stream = s; g_free_clean = false; }
void set_stream_synced() { g_cur_stream = nullptr; g_free_clean = true; }

dbl_status order_after_caller(dbl_graph *g) {
    DBL_CUDA(cudaEventRecord(g->ev_in, cudaStreamLegacy));
    DBL_CUDA(cudaStreamWaitEvent(g->stream, g->ev_in, 0));
    return DBL_OK;
}

static size_t size_class(size_t n) {
    if (n <= 4096) {
        size_t c = 256;
        while (c < n) c <<= 1;
        return c;
    }
    size_t oct = 1;
    while ((oct << 1) <= n) oct <<= 1;           // oct <= n < 2 oct
    const size_t step = oct / 8;
    return (n + step - 1) / step * step;
}

cudaError_t pool_alloc(void **p, size_t *bytes, int *device) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t c = size_class(*bytes);
    PoolBlock blk{nullptr, nullptr, false};
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        auto it = g_pool.find({dev, c});
        if (it != g_pool.end() && !it->second.empty()) {
            auto &v = it->second;
            size_t pick = v.size() - 1;
            for (size_t i = 0; i < v.size(); ++i)
                if (v[i].s == g_cur_stream && g_cur_stream) { pick = i; break; }
            blk = v[pick];
            v.erase(v.begin() + pick);
        }
    }
    if (blk.p) {
        if (!blk.clean && (blk.s != g_cur_stream || !blk.s)) {
            if (blk.s) cudaStreamSynchronize(blk.s); else cudaDeviceSynchronize();
        }
        *p = blk.p;
        *bytes = c;
        *device = dev;
        return cudaSuccess;
    }
    cudaError_t e = cudaMalloc(p, c);
    if (e == cudaErrorMemoryAllocation) {  // give cached blocks back and retry once
        cudaGetLastError();
        pool_trim();
        e = cudaMalloc(p, c);
    }
    if (e != cudaSuccess) return e;
    *bytes = c;
    *device = dev;
    return cudaSuccess;
}

void pool_forget_stream(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (auto &kv : g_pool)
        for (auto &b : kv.second)
            if (b.s == st) b.s = nullptr;
}

void pool_free(void *p, size_t bytes, int device) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool[{device, bytes}].push_back(PoolBlock{p, g_cur_stream, g_free_clean});
}

void pool_trim() {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : g_pool) {
        cudaSetDevice(kv.first.first);
        cudaDeviceSynchronize();
        for (auto &b : kv.second) cudaFree(b.p);
        kv.second.clear();
    }
    cudaSetDevice(cur);
}

static auto g_trace_t0 = std::chrono::steady_clock::now();

void trace(const char *what, cudaStream_t s) {
    if (!DBL_TRACE) return;
    if (DBL_TRACE == 1) cudaStreamSynchronize(s);   // 2: host enqueue times only
    auto now = std::chrono::steady_clock::now();
    double us = std::chrono::duration<double, std::micro>(now - g_trace_t0).count();
    std::fprintf(stderr, "[dbl] %-28s +%9.1f us\n", what, us);
    g_trace_t0 = std::chrono::steady_clock::now();
}

dbl_status cuda_fail(cudaError_t e, const char *what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? DBL_E_OOM : DBL_E_CUDA;
}

// Occupancy cache: the dynamic shared-memory opt-in is a per-device function
// attribute, and handles on different devices may be driven from different
// host threads (dbl_query_multi), so both the attribute and the occupancy
// are cached per (device, kernel, threads, smem) under a mutex.
static std::mutex g_occ_mu;
static std::map<std::tuple<int, const void *, int, size_t>, int> g_occ;

dbl_status kernel_occupancy(const void *fn, int threads, size_t smem, int *bps) {
    int dev = 0;
    DBL_CUDA(cudaGetDevice(&dev));
    const auto key = std::make_tuple(dev, fn, threads, smem);
    {
        std::lock_guard<std::mutex> lk(g_occ_mu);
        auto it = g_occ.find(key);
        if (it != g_occ.end()) { *bps = it->second; return DBL_OK; }
    }
    if (smem > 48 * 1024)
        DBL_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int b = 0;
    DBL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem));
    if (b < 1) b = 1;
    std::lock_guard<std::mutex> lk(g_occ_mu);
    g_occ[key] = b;
    *bps = b;
    return DBL_OK;
}

dbl_status make_override(dbl_graph *g, const uint32_t *ids, const uint32_t *buckets, uint32_t cnt,
                         DevBuf &ovr);

static int grid_for(uint64_t work, int threads = 256, int cap = 148 * 16) {
    uint64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > (uint64_t)cap) b = cap;
    return (int)b;
}

__global__ void certified_kernel(const uint64_t *__restrict__ rec, uint32_t rs, uint32_t H, uint32_t wdl,
                                 const uint64_t *__restrict__ keys, uint64_t count,
                                 unsigned long long *out, const uint64_t *__restrict__ valid_dev = nullptr,
                                 const unsigned long long *__restrict__ abort_dev = nullptr) {
    if (valid_dev) count = (abort_dev && *abort_dev) ? 0ull : min(count, *valid_dev);
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const uint64_t *ru = rec + (k >> 32) * rs, *rv = rec + (uint32_t)k * (uint64_t)rs;
        uint64_t acc = 0;
        for (uint32_t w = 0; w < wdl; ++w) acc |= ru[H + w] & rv[w];  // dl_out[u] & dl_in[v]
        c += acc != 0;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// keys = (u << shift) | v; shift = 32 for the canonical layout, or the
// vertex-id width so that a radix sort needs 2 * shift bits, not 32 + shift
__global__ void pack_pairs_kernel(const uint32_t *__restrict__ u, const uint32_t *__restrict__ v,
                                  uint64_t count, uint32_t n, uint64_t *__restrict__ keys,
                                  unsigned long long *err, uint32_t shift = 32) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a = u[i], b = v[i];
        if (a >= n || b >= n) { atomicOr(err, 1ull); a = 0; b = 0; }
        keys[i] = ((uint64_t)a << shift) | b;
    }
}

// (u << shift | v) -> (u << 32 | v), in place
__global__ void widen_keys_kernel(uint64_t *__restrict__ keys, uint64_t count, uint32_t shift,
                                  const uint64_t *__restrict__ valid_dev = nullptr) {
    if (valid_dev) count = min(count, *valid_dev);
    const uint64_t mask = (1ull << shift) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        keys[i] = ((k >> shift) << 32) | (k & mask);
    }
}

// family f of a record: (word offset within record, words)
static void family_span(const dbl_index *idx, int f, uint32_t &off, uint32_t &w) {
    const uint32_t H = idx->wdl + idx->wbl;
    switch (f) {
    case 0: off = 0; w = idx->wdl; break;                 // dl_in
    case 1: off = H; w = idx->wdl; break;                 // dl_out
    case 2: off = idx->wdl; w = idx->wbl; break;          // bl_in
    default: off = H + idx->wdl; w = idx->wbl; break;     // bl_out
    }
}

__global__ void gather_family_kernel(const uint64_t *__restrict__ rec, uint32_t rs, uint32_t off, uint32_t w,
                                     uint32_t n, uint64_t *__restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)n * w;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = rec[(i / w) * rs + off + i % w];
}

__global__ void scatter_family_kernel(uint64_t *__restrict__ rec, uint32_t rs, uint32_t off, uint32_t w,
                                      uint32_t n, const uint64_t *__restrict__ in) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)n * w;
         i += (uint64_t)gridDim.x * blockDim.x)
        rec[(i / w) * rs + off + i % w] = in[i];
}

// label words only: a record's pad words past 2H are unspecified
__global__ void diff_kernel(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b, uint64_t count,
                            uint32_t rs, uint32_t rw, unsigned long long *out) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        c |= (i % rs < rw) && a[i] != b[i];
    if (__any_sync(FULL, c) && (threadIdx.x & 31) == 0) atomicOr(out, 1ull);
}

__global__ void fill_tail_kernel(uint32_t *__restrict__ ptr, uint32_t from, uint32_t to) {
    const uint32_t val = ptr[from - 1];
    for (uint32_t i = from + blockIdx.x * blockDim.x + threadIdx.x; i < to; i += gridDim.x * blockDim.x)
        ptr[i] = val;
}

}  // namespace dbl

using namespace dbl;

extern "C" const char *dbl_last_error(void) { return g_last_error.c_str(); }
extern "C" int dbl_version(void) { return 1; }
extern "C" uint64_t dbl_kernel_launches(void) { return g_launches.load(); }
extern "C" dbl_status dbl_release_cached_memory(void) {
    ServeBlock no_service_;   // no per-call service runs during this call
    pool_trim();
    return DBL_OK;
}

static dbl_status check_pair(const dbl_index *idx, const dbl_graph *g) {
    if (!idx || !g) { set_error("null handle"); return DBL_E_ARG; }
    if (idx->n != g->n) {
        set_error("graph has " + std::to_string(g->n) + " vertices but index has " + std::to_string(idx->n));
        return DBL_E_MISMATCH;
    }
    return DBL_OK;
}

static dbl_status alloc_index(const dbl_graph *g, const dbl_config *cfg, dbl_index **out) {
    if (cfg->k > g->n) {
        set_error("k=" + std::to_string(cfg->k) + " exceeds vertex count " + std::to_string(g->n));
        return DBL_E_CONFIG;
    }
    if (cfg->k_prime < 1) { set_error("k_prime must be >= 1"); return DBL_E_CONFIG; }
    if (cfg->strategy < 0 || cfg->strategy > 3) { set_error("unknown landmark strategy"); return DBL_E_CONFIG; }
    dbl_index *idx = new dbl_index();
    idx->device = g->device;
    idx->n = g->n;
    idx->cfg = *cfg;
    idx->wdl = (cfg->k + 63) / 64;
    idx->wbl = (cfg->k_prime + 63) / 64;
    idx->rw = 2 * (idx->wdl + idx->wbl);
    idx->rs = rec_stride(idx->wdl + idx->wbl);
    if (idx->wdl > 16 || idx->wbl > 16 || idx->rw > 64) {
        delete idx;
        set_error("label widths above 1024 bits are not supported");
        return DBL_E_CONFIG;
    }
    dbl_status s;
    if ((s = idx->rec.ensure((size_t)g->n * idx->rs * 8 + 16)) || (s = idx->landmarks.ensure((size_t)cfg->k * 4 + 4)) ||
        (s = idx->leaf_flags.ensure((size_t)g->n + 16)) || (s = idx->bucket.ensure((size_t)g->n * 4 + 16))) {
        dbl_index_free(idx);
        return s;
    }
    // pad words (rs > rw) are zeroed by whichever pass seeds the records
    // (prep_kernel for a build, seed_records_kernel otherwise) and never
    // written again; grown records are zero-filled
    *out = idx;
    return DBL_OK;
}

static dbl_status index_create(const dbl_graph *gc, const dbl_config *cfg, const uint32_t *landmarks,
                                      const uint8_t *leaf_flags, const uint32_t *bucket,
                                      const uint32_t *ovr_ids, const uint32_t *ovr_buckets, uint32_t n_ovr,
                                      dbl_index **out, bool seed = true) {
    if (!gc || !cfg || !out) { set_error("null argument"); return DBL_E_ARG; }
    *out = nullptr;
    dbl_graph *g = const_cast<dbl_graph *>(gc);
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    if (landmarks && cfg->k) {  // LandmarkSet.of + _check_vertex (labels.py:59-63, 279-283)
        std::vector<uint32_t> seen(landmarks, landmarks + cfg->k);
        for (uint32_t i = 0; i < cfg->k; ++i)
            if (landmarks[i] >= g->n) {
                set_error("vertex " + std::to_string(landmarks[i]) + " outside [0, " + std::to_string(g->n) + ")");
                return DBL_E_VERTEX_RANGE;
            }
        std::sort(seen.begin(), seen.end());
        if (std::adjacent_find(seen.begin(), seen.end()) != seen.end()) {
            set_error("landmark vertices must be distinct");
            return DBL_E_CONFIG;
        }
    }
    dbl_index *idx = nullptr;
    trace("build: enter", g->stream);
    dbl_status s = alloc_index(g, cfg, &idx);
    if (s) return s;
    trace("build: alloc", g->stream);
    auto fail = [&](dbl_status st) { dbl_index_free(idx); return st; };
    if (cfg->k) {
        if (landmarks) {
            DBL_CUDA(cudaMemcpyAsync(idx->landmarks.p, landmarks, (size_t)cfg->k * 4, cudaMemcpyHostToDevice, g->stream));
        } else if (!seed) {
            idx->sel_landmarks = true;   // selected on the device by the build's prep pass
        } else if ((s = select_landmarks_dev(g, cfg->k, cfg->strategy, idx->landmarks.as<uint32_t>()))) {
            return fail(s);
        }
    }
    trace("build: landmarks", g->stream);
    if (g->n) {
        if (leaf_flags && bucket) {
            DBL_CUDA(cudaMemcpyAsync(idx->leaf_flags.p, leaf_flags, g->n, cudaMemcpyHostToDevice, g->stream));
            DBL_CUDA(cudaMemcpyAsync(idx->bucket.p, bucket, (size_t)g->n * 4, cudaMemcpyHostToDevice, g->stream));
        } else if (!seed) {
            // leaves are selected by the build's prep pass (override errors
            // are reported when the build finishes)
            if (cfg->k_prime < 1) { set_error("k_prime must be >= 1"); return fail(DBL_E_CONFIG); }
            if (ovr_ids && n_ovr && (s = make_override(g, ovr_ids, ovr_buckets, n_ovr, idx->ovr))) return fail(s);
            idx->sel_leaves = true;
        } else {
            DevBuf ovr;
            const uint32_t *dovr = nullptr;
            if (ovr_ids && n_ovr) {
                if ((s = make_override(g, ovr_ids, ovr_buckets, n_ovr, ovr))) { ovr.release(); return fail(s); }
                dovr = ovr.as<uint32_t>();
            }
            s = select_leaves_dev(g, cfg->leaf_threshold, cfg->k_prime, cfg->hash_seed, dovr,
                                  idx->leaf_flags.as<uint8_t>(), idx->bucket.as<uint32_t>());
            ovr.release();
            if (s) return fail(s);
        }
    }
    trace("build: leaves", g->stream);
    if (seed && (s = index_seed_records(g, idx, ~0ull))) return fail(s);
    *out = idx;
    return DBL_OK;
}

extern "C" dbl_status dbl_index_create(const dbl_graph *gc, const dbl_config *cfg, const uint32_t *landmarks,
                                       const uint8_t *leaf_flags, const uint32_t *bucket, const uint32_t *ovr_ids,
                                       const uint32_t *ovr_buckets, uint32_t n_ovr, dbl_index **out) {
    ServeBlock no_service_;   // no per-call service runs during this call
    return index_create(gc, cfg, landmarks, leaf_flags, bucket, ovr_ids, ovr_buckets, n_ovr, out);
}

extern "C" dbl_status dbl_index_build(const dbl_graph *gc, const dbl_config *cfg, const uint32_t *landmarks,
                                      const uint8_t *leaf_flags, const uint32_t *bucket,
                                      const uint32_t *ovr_ids, const uint32_t *ovr_buckets, uint32_t n_ovr,
                                      dbl_index **out) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (out) *out = nullptr;
    dbl_index *idx = nullptr;
    dbl_status s = index_create(gc, cfg, landmarks, leaf_flags, bucket, ovr_ids, ovr_buckets, n_ovr, &idx, false);
    if (s) return s;
    // the digest is part of the built index (its pass is inside the build's time)
    if ((s = run_build(const_cast<dbl_graph *>(gc), idx, nullptr, 0)) ||
        (s = digest_refresh(idx, const_cast<dbl_graph *>(gc)))) {
        dbl_index_free(idx);
        return s;
    }
    *out = idx;
    return DBL_OK;
}

extern "C" dbl_status dbl_index_rebuild(const dbl_graph *gc, dbl_index *idx) {
    ServeBlock no_service_;   // no per-call service runs during this call
    dbl_status s = check_pair(idx, gc);
    if (s) return s;
    dbl_graph *g = const_cast<dbl_graph *>(gc);
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    ++idx->version;
    if ((s = run_build(g, idx, nullptr, 0))) return s;
    return digest_refresh(idx, g);
}

extern "C" dbl_status dbl_index_build_words(const dbl_graph *gc, dbl_index *idx, const uint32_t *words,
                                            uint32_t nwords) {
    ServeBlock no_service_;   // no per-call service runs during this call
    dbl_status s = check_pair(idx, gc);
    if (s) return s;
    for (uint32_t i = 0; i < nwords; ++i)
        if (words[i] >= idx->rw) { set_error("record word out of range"); return DBL_E_ARG; }
    dbl_graph *g = const_cast<dbl_graph *>(gc);
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    ++idx->version;
    return run_build(g, idx, words, nwords);
}

extern "C" dbl_status dbl_index_free(dbl_index *idx) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx) return DBL_OK;
    cudaSetDevice(idx->device);
    cudaDeviceSynchronize();
    set_stream_synced();
    idx->rec.release();
    idx->digest.release();
    idx->landmarks.release();
    idx->leaf_flags.release();
    idx->bucket.release();
    idx->ovr.release();
    idx->dmask.release();
    idx->sccmask.release();
    delete idx;
    return DBL_OK;
}

extern "C" dbl_status dbl_index_info(const dbl_index *idx, uint32_t *n, dbl_config *cfg) {
    if (!idx) { set_error("null index"); return DBL_E_ARG; }
    if (n) *n = idx->n;
    if (cfg) *cfg = idx->cfg;
    return DBL_OK;
}

extern "C" dbl_status dbl_index_metadata(const dbl_index *idx, uint32_t *landmarks, uint8_t *leaf_flags,
                                         uint32_t *bucket) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx) { set_error("null index"); return DBL_E_ARG; }
    DBL_CUDA(cudaSetDevice(idx->device));
    set_stream(nullptr);
    if (landmarks && idx->cfg.k) DBL_CUDA(cudaMemcpy(landmarks, idx->landmarks.p, (size_t)idx->cfg.k * 4, cudaMemcpyDeviceToHost));
    if (leaf_flags && idx->n) DBL_CUDA(cudaMemcpy(leaf_flags, idx->leaf_flags.p, idx->n, cudaMemcpyDeviceToHost));
    if (bucket && idx->n) DBL_CUDA(cudaMemcpy(bucket, idx->bucket.p, (size_t)idx->n * 4, cudaMemcpyDeviceToHost));
    return DBL_OK;
}

extern "C" dbl_status dbl_index_export(const dbl_index *idx, uint64_t *dl_in, uint64_t *dl_out, uint64_t *bl_in,
                                       uint64_t *bl_out) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx) { set_error("null index"); return DBL_E_ARG; }
    DBL_CUDA(cudaSetDevice(idx->device));
    set_stream(nullptr);
    uint64_t *outs[4] = {dl_in, dl_out, bl_in, bl_out};
    DevBuf tmp;
    for (int f = 0; f < 4; ++f) {
        uint32_t off, w;
        family_span(idx, f, off, w);
        if (!outs[f] || !w || !idx->n) continue;
        const uint64_t cnt = (uint64_t)idx->n * w;
        dbl_status s = tmp.ensure(cnt * 8);
        if (s) return s;
        gather_family_kernel<<<grid_for(cnt), 256>>>(idx->rec.as<uint64_t>(), idx->rs, off, w, idx->n,
                                                     tmp.as<uint64_t>());
        DBL_LAUNCHED();
        cudaError_t e = cudaMemcpy(outs[f], tmp.p, cnt * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { tmp.release(); return cuda_fail(e, "export labels"); }
    }
    tmp.release();
    return DBL_OK;
}

extern "C" dbl_status dbl_index_import(dbl_index *idx, const uint64_t *dl_in, const uint64_t *dl_out,
                                       const uint64_t *bl_in, const uint64_t *bl_out) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx) { set_error("null index"); return DBL_E_ARG; }
    DBL_CUDA(cudaSetDevice(idx->device));
    set_stream(nullptr);
    ++idx->version;
    const uint64_t *ins[4] = {dl_in, dl_out, bl_in, bl_out};
    DevBuf tmp;
    for (int f = 0; f < 4; ++f) {
        uint32_t off, w;
        family_span(idx, f, off, w);
        if (!ins[f] || !w || !idx->n) continue;
        const uint64_t cnt = (uint64_t)idx->n * w;
        dbl_status s = tmp.ensure(cnt * 8);
        if (s) return s;
        cudaError_t e = cudaMemcpy(tmp.p, ins[f], cnt * 8, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { tmp.release(); return cuda_fail(e, "import labels"); }
        scatter_family_kernel<<<grid_for(cnt), 256>>>(idx->rec.as<uint64_t>(), idx->rs, off, w, idx->n,
                                                      tmp.as<uint64_t>());
        DBL_LAUNCHED();
    }
    cudaError_t e = cudaDeviceSynchronize();
    tmp.release();
    if (e != cudaSuccess) return cuda_fail(e, "import labels");
    return DBL_OK;
}

extern "C" dbl_status dbl_index_equal(const dbl_index *a, const dbl_index *b, int *out_equal) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!a || !b || !out_equal) { set_error("null argument"); return DBL_E_ARG; }
    *out_equal = 0;
    if (a->n != b->n || a->cfg.k != b->cfg.k || a->cfg.k_prime != b->cfg.k_prime) return DBL_OK;
    if (a->device != b->device) { set_error("indexes live on different devices"); return DBL_E_ARG; }
    DBL_CUDA(cudaSetDevice(a->device));
    set_stream(nullptr);
    DevBuf flag;
    dbl_status s = flag.ensure(8);
    if (s) return s;
    cudaMemset(flag.p, 0, 8);
    const uint64_t cnt = (uint64_t)a->n * a->rs;
    if (cnt) {
        diff_kernel<<<grid_for(cnt), 256>>>(a->rec.as<uint64_t>(), b->rec.as<uint64_t>(), cnt, a->rs,
                                            2 * (a->wdl + a->wbl), flag.as<unsigned long long>());
        DBL_LAUNCHED();
    }
    unsigned long long h = 1;
    cudaError_t e = cudaMemcpy(&h, flag.p, 8, cudaMemcpyDeviceToHost);
    flag.release();
    if (e != cudaSuccess) return cuda_fail(e, "index_equal");
    *out_equal = h == 0;
    return DBL_OK;
}

static dbl_status grow_buf(DevBuf &b, size_t old_bytes, size_t new_bytes, int fill) {
    DevBuf nb;
    dbl_status s = nb.ensure(new_bytes);
    if (s) return s;
    if (old_bytes) DBL_CUDA(cudaMemcpy(nb.p, b.p, old_bytes, cudaMemcpyDeviceToDevice));
    if (new_bytes > old_bytes) DBL_CUDA(cudaMemset(nb.as<char>() + old_bytes, fill, new_bytes - old_bytes));
    b.release();
    b = nb;
    return DBL_OK;
}

extern "C" dbl_status dbl_index_grow(dbl_index *idx, uint32_t n) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx) { set_error("null index"); return DBL_E_ARG; }
    if (n < idx->n) { set_error("index cannot shrink"); return DBL_E_CONFIG; }
    if (n == idx->n) return DBL_OK;
    DBL_CUDA(cudaSetDevice(idx->device));
    set_stream(nullptr);
    dbl_status s;
    if ((s = grow_buf(idx->rec, (size_t)idx->n * idx->rs * 8, (size_t)n * idx->rs * 8 + 16, 0)) ||
        (s = grow_buf(idx->leaf_flags, idx->n, (size_t)n + 16, 0)) ||
        (s = grow_buf(idx->bucket, (size_t)idx->n * 4, (size_t)n * 4 + 16, 0)))
        return s;
    idx->n = n;
    ++idx->version;
    return DBL_OK;
}

extern "C" dbl_status dbl_graph_add_vertices(dbl_graph *g, uint32_t count) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!g) { set_error("null graph"); return DBL_E_ARG; }
    if (!count) return DBL_OK;
    if ((uint64_t)g->n + count >= 0xffffffffull) { set_error("vertex count overflow"); return DBL_E_CONFIG; }
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    const uint32_t n0 = g->n, n1 = n0 + count;
    DevBuf *ptrs[4] = {&g->fptr, &g->rptr, &g->dfptr, &g->drptr};
    for (int i = 0; i < 4; ++i) {
        if (i >= 2 && !g->m_delta) { ptrs[i]->release(); continue; }
        dbl_status s = grow_buf(*ptrs[i], ((size_t)n0 + 1) * 4, ((size_t)n1 + 1) * 4, 0);
        if (s) return s;
        fill_tail_kernel<<<grid_for(count), 256>>>(ptrs[i]->as<uint32_t>(), n0 + 1, n1 + 1);
        DBL_LAUNCHED();
    }
    DBL_CUDA(cudaDeviceSynchronize());
    g->n = n1;
    ++g->topo_version;
    for (int d = 0; d < 2; ++d) g->stamp[d].release();
    g->changed_bits.release();
    return graph_ensure_traversal(g);
}

extern "C" dbl_status dbl_index_records(const dbl_index *idx, uint64_t **dev_records, uint32_t *wpr) {
    if (!idx) { set_error("null index"); return DBL_E_ARG; }
    if (dev_records) *dev_records = idx->rec.as<uint64_t>();
    if (wpr) *wpr = idx->rs;
    return DBL_OK;
}

extern "C" dbl_status dbl_graph_instrument(dbl_graph *g, int on) {
    if (!g) { set_error("null graph"); return DBL_E_ARG; }
    g->instrument = on != 0;
    return DBL_OK;
}

// Executed work of the last build on g (bench roofline: bytes actually moved).
extern "C" dbl_status dbl_build_work_stats(const dbl_graph *g, dbl_build_work *out) {
    if (!g || !out) { set_error("null argument"); return DBL_E_ARG; }
    DBL_CUDA(cudaSetDevice(g->device));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    dbl_build_work w{};
    w.n = g->n;
    w.m = g->m_base + g->m_delta;
    w.record_bytes = 8 * g->last_build.rs;
    w.flags = g->last_build.flags;
    w.fix_levels = g->last_build.fix_levels;
    w.fix_runs = g->last_build.fix_runs;
    w.fix_items = g->last_build.fix_items;
    w.fix_edges = g->last_build.fix_edges;
    if (g->reach_work) {
        unsigned long long c[5];
        unsigned int st[6];
        DBL_CUDA(cudaMemcpy(c, g->reach_work, sizeof(c), cudaMemcpyDeviceToHost));
        DBL_CUDA(cudaMemcpy(st, g->reach_chg, sizeof(st), cudaMemcpyDeviceToHost));
        w.bu_tests = c[0];
        w.bu_probes = c[1];
        w.td_vertices = c[2];
        w.td_edges = c[3];
        w.union_records = c[4];
        w.steps = st[4];
        w.sweeps = st[5];
        if (st[3]) w.flags |= 8u;
    }
    *out = w;
    return DBL_OK;
}

// ---------------------------------------------------------------- queries --

#ifndef DBL_PIPE_CHUNK_LOG2
#define DBL_PIPE_CHUNK_LOG2 18   // pairs per chunk of the copy pipeline (log2)
#endif
#ifndef DBL_PINNED_DMA
#define DBL_PINNED_DMA 0         // > 0: pinned batches of >= 2^DBL_PINNED_DMA pairs take the copy pipeline
#endif

// Host-memory batches are pipelined in chunks: the H2D copy of chunk i+1
// (copy stream), the query kernels of chunk i (engine stream) and the D2H copy
// of chunk i-1 (second copy stream) overlap, so PCIe traffic in both
// directions hides the device work.
static dbl_status query_host_pipelined(const dbl_index *idx, dbl_graph *g, const uint32_t *u, const uint32_t *v,
                                       uint64_t count, uint32_t flags, uint8_t *codes, uint32_t *visited) {
    dbl_status s;
    const uint64_t cpad = (count + 63) & ~63ull;
    if ((s = g->q_in.ensure(cpad * 8 + 64)) || (s = g->q_codes.ensure(count + 64)) ||
        (visited && (s = g->q_vis.ensure(count * 4 + 64))) || (s = g->q_errs.ensure(64 * 4)))
        return s;
    if (!g->cstream[0]) {
        DBL_CUDA(cudaStreamCreateWithFlags(&g->cstream[0], cudaStreamNonBlocking));
        DBL_CUDA(cudaStreamCreateWithFlags(&g->cstream[1], cudaStreamNonBlocking));
        for (auto &e : g->cev) DBL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const uint64_t target = 1ull << DBL_PIPE_CHUNK_LOG2;
    uint64_t nch = (count + target - 1) / target;
    if (nch < 1) nch = 1;
    if (nch > 16) nch = 16;
    uint64_t csz = (count + nch - 1) / nch;
    csz = (csz + 127) & ~127ull;
    nch = (count + csz - 1) / csz;
    uint32_t *bu = g->q_in.as<uint32_t>(), *bv = bu + cpad;
    uint8_t *dc = g->q_codes.as<uint8_t>();
    uint32_t *dvis = visited ? g->q_vis.as<uint32_t>() : nullptr;
    uint32_t *errs = g->q_errs.as<uint32_t>();
    DBL_CUDA(cudaMemsetAsync(errs, 0, 64 * 4, g->stream));
    DBL_CUDA(cudaEventRecord(g->cev[32], g->stream));            // errs cleared
    DBL_CUDA(cudaStreamWaitEvent(g->cstream[1], g->cev[32], 0));
    for (uint64_t i = 0; i < nch; ++i) {
        const uint64_t lo = i * csz, hi = lo + csz < count ? lo + csz : count, c = hi - lo;
        DBL_CUDA(cudaMemcpyAsync(bu + lo, u + lo, c * 4, cudaMemcpyHostToDevice, g->cstream[0]));
        DBL_CUDA(cudaMemcpyAsync(bv + lo, v + lo, c * 4, cudaMemcpyHostToDevice, g->cstream[0]));
        DBL_CUDA(cudaEventRecord(g->cev[i], g->cstream[0]));
        DBL_CUDA(cudaStreamWaitEvent(g->stream, g->cev[i], 0));
        if ((s = run_query(idx, g, bu + lo, bv + lo, c, flags, dc + lo, dvis ? dvis + lo : nullptr))) return s;
        if ((s = query_err_to(g, errs + 4 * i))) return s;
        DBL_CUDA(cudaEventRecord(g->cev[16 + i], g->stream));
        DBL_CUDA(cudaStreamWaitEvent(g->cstream[1], g->cev[16 + i], 0));
        DBL_CUDA(cudaMemcpyAsync(codes + lo, dc + lo, c, cudaMemcpyDeviceToHost, g->cstream[1]));
        if (visited) DBL_CUDA(cudaMemcpyAsync(visited + lo, dvis + lo, c * 4, cudaMemcpyDeviceToHost, g->cstream[1]));
    }
    uint32_t herr[64];
    DBL_CUDA(cudaMemcpyAsync(herr, errs, 64 * 4, cudaMemcpyDeviceToHost, g->cstream[1]));
    DBL_CUDA(cudaStreamSynchronize(g->cstream[1]));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    bool dense = false;
    for (uint64_t i = 0; i < nch; ++i) {
        if (herr[4 * i]) { set_error("query vertex outside [0, n)"); return DBL_E_VERTEX_RANGE; }
        dense |= chunk_needs_dense(herr + 4 * i);
    }
    if (dense) {   // some chunk needed the dense BFS workspace: allocate it, run again
        if ((s = ensure_dense(idx, g))) return s;
        return query_host_pipelined(idx, g, u, v, count, flags, codes, visited);
    }
    return DBL_OK;
}

// Small pageable host batches: the pairs are copied into a pinned staging
// buffer of the graph and read by the query kernel over PCIe (zero-copy),
// which also writes the codes there; one launch and one stream sync instead
// of the copy pipeline's seven operations (a single query() call).
constexpr uint64_t STAGE_MAX = 1ull << 16;
#ifndef DBL_STAGE_ALL
#define DBL_STAGE_ALL 1   // 1: large pageable batches are staged too (parallel host copies), 0: copy pipeline
#endif

// memcpy split over host threads for large buffers (pageable <-> pinned
// staging runs at one core's copy bandwidth otherwise)
static void par_memcpy(void *dst, const void *src, size_t bytes) {
    constexpr size_t MIN_PART = 1u << 20;
    const unsigned hw = std::thread::hardware_concurrency();
    size_t parts = bytes / MIN_PART;
    if (parts > 8) parts = 8;
    if (hw && parts > hw) parts = hw;
    if (parts < 2) { std::memcpy(dst, src, bytes); return; }
    const size_t chunk = (bytes / parts + 63) & ~(size_t)63;
    std::vector<std::thread> ts;
    ts.reserve(parts - 1);
    for (size_t i = 1; i < parts; ++i) {
        const size_t lo = i * chunk;
        if (lo >= bytes) break;
        const size_t len = lo + chunk <= bytes ? chunk : bytes - lo;
        ts.emplace_back([=] { std::memcpy((char *)dst + lo, (const char *)src + lo, len); });
    }
    std::memcpy(dst, src, chunk < bytes ? chunk : bytes);
    for (auto &t : ts) t.join();
}

static dbl_status query_host_staged(const dbl_index *idx, dbl_graph *g, const uint32_t *u, const uint32_t *v,
                                    uint64_t count, uint32_t flags, uint8_t *codes, uint32_t *visited) {
    dbl_status s;
    const uint64_t cpad = (count + 63) & ~63ull;
    if ((s = g->q_stage.ensure(cpad * 13 + 256))) return s;
    uint32_t *su = reinterpret_cast<uint32_t *>(g->q_stage.p), *sv = su + cpad;
    uint32_t *svis = sv + cpad;
    uint8_t *sc = reinterpret_cast<uint8_t *>(svis + cpad);
    par_memcpy(su, u, count * 4);
    par_memcpy(sv, v, count * 4);
    if ((s = run_query(idx, g, su, sv, count, flags, sc, visited ? svis : nullptr, true, true))) return s;
    uint32_t err = 0;
    bool dense = false;
    if ((s = query_finish(g, &err, &dense))) return s;
    if (err) { set_error("query vertex outside [0, n)"); return DBL_E_VERTEX_RANGE; }
    if (dense) {
        if ((s = ensure_dense(idx, g))) return s;
        return query_host_staged(idx, g, u, v, count, flags, codes, visited);
    }
    par_memcpy(codes, sc, count);
    if (visited) par_memcpy(visited, svis, count * 4);
    return DBL_OK;
}

static dbl_status query_impl(const dbl_index *idx, const dbl_graph *gc, const uint32_t *u, const uint32_t *v,
                             uint64_t count, uint32_t flags, uint8_t *codes, uint32_t *visited, dbl_mem mem,
                             bool sync) {
    dbl_status s = check_pair(idx, gc);
    if (s) return s;
    if (count && (!u || !v || !codes)) { set_error("null argument"); return DBL_E_ARG; }
    dbl_graph *g = const_cast<dbl_graph *>(gc);
    if (count == 1 && mem == DBL_MEM_HOST && sync) {
        // a single query() call: the resident service warp answers it
        // (query.cu K6s), no launch or stream sync per call
        const uint32_t hu = u[0], hv = v[0];
        if (hu >= g->n || hv >= g->n) { set_error("query vertex outside [0, n)"); return DBL_E_VERTEX_RANGE; }
        bool served = false;
        if ((s = serve_query(idx, g, hu, hv, flags, codes, visited, &served))) return s;
        if (served) return DBL_OK;
    }
    ServeBlock no_service_;   // batch path: no per-call service runs during it
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    if (mem == DBL_MEM_HOST && count) {
        // Page-locked host buffers are read and written by the query kernels
        // directly over PCIe (zero-copy): the transfer streams under the
        // label checks instead of being staged.  Pageable memory goes
        // through the chunked copy pipeline.
        const void *ptrs[4] = {u, v, codes, visited};
        void *dptr[4] = {nullptr, nullptr, nullptr, nullptr};
        bool pinned = true;
        for (int i = 0; i < 4 && pinned; ++i) {
            if (!ptrs[i]) continue;
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, ptrs[i]) != cudaSuccess || at.type != cudaMemoryTypeHost ||
                !at.devicePointer) {
                cudaGetLastError();
                pinned = false;
            } else {
                dptr[i] = at.devicePointer;
            }
        }
        if (pinned && DBL_PINNED_DMA && count >= (1ull << DBL_PINNED_DMA))
            return query_host_pipelined(idx, g, u, v, count, flags, codes, visited);
        if (!pinned)
            return (DBL_STAGE_ALL || count <= STAGE_MAX)
                       ? query_host_staged(idx, g, u, v, count, flags, codes, visited)
                       : query_host_pipelined(idx, g, u, v, count, flags, codes, visited);
        if ((s = run_query(idx, g, (const uint32_t *)dptr[0], (const uint32_t *)dptr[1], count, flags,
                           (uint8_t *)dptr[2], (uint32_t *)dptr[3], sync, true)))
            return s;
    } else {
        // the synchronous call orders itself after the caller's default-stream
        // work; dbl_query_async is stream-ordered only (dbl_b200.h)
        if (count && sync && (s = order_after_caller(g))) return s;
        if ((s = run_query(idx, g, u, v, count, flags, codes, visited, sync))) return s;
    }
    if (!sync) return DBL_OK;
    uint32_t err = 0;
    bool dense = false;
    if ((s = query_finish(g, &err, &dense))) return s;
    if (err) { set_error("query vertex outside [0, n)"); return DBL_E_VERTEX_RANGE; }
    if (dense) {   // the batch needed the dense BFS workspace: allocate it, run again
        if ((s = ensure_dense(idx, g))) return s;
        return query_impl(idx, gc, u, v, count, flags, codes, visited, mem, sync);
    }
    return DBL_OK;
}

extern "C" dbl_status dbl_query(const dbl_index *idx, const dbl_graph *g, const uint32_t *u, const uint32_t *v,
                                uint64_t count, uint32_t flags, uint8_t *codes, uint32_t *visited, dbl_mem mem) {
    return query_impl(idx, g, u, v, count, flags, codes, visited, mem, true);
}

// query() for one pair with scalar arguments (the per-call path):
// out[0] = AnsweredBy code, out[1] = visited.
extern "C" dbl_status dbl_query_one(const dbl_index *idx, const dbl_graph *g, uint32_t u, uint32_t v,
                                    uint32_t flags, uint32_t *out) {
    if (!out) { set_error("null argument"); return DBL_E_ARG; }
    uint8_t code = 0;
    uint32_t visited = 0;
    dbl_status s = query_impl(idx, g, &u, &v, 1, flags, &code, &visited, DBL_MEM_HOST, true);
    if (s) return s;
    out[0] = code;
    out[1] = visited;
    return DBL_OK;
}

extern "C" dbl_status dbl_query_async(const dbl_index *idx, const dbl_graph *g, const uint32_t *u,
                                      const uint32_t *v, uint64_t count, uint32_t flags, uint8_t *codes,
                                      uint32_t *visited) {
    ServeBlock no_service_;   // no per-call service runs during this call
    return query_impl(idx, g, u, v, count, flags, codes, visited, DBL_MEM_DEVICE, false);
}

// One batch split across several devices: contiguous,
// order-preserving slices as in the reference's worker pool
// (queries.py:224-232: chunk = ceil(count / parts)), each answered on its
// own handle pair from one host thread per device, so the slices' transfers
// and kernels run concurrently.  The replicas must be identical (same graph
// and index built on every device).  Host batches: every slice crosses PCIe
// to its own GPU.  Device batches (all buffers on one GPU): the other GPUs
// read their slices and write their codes over NVLink by peer access.
extern "C" dbl_status dbl_query_multi(const dbl_index *const *idx, const dbl_graph *const *g, uint32_t ndev,
                                      const uint32_t *u, const uint32_t *v, uint64_t count, uint32_t flags,
                                      uint8_t *codes, uint32_t *visited, dbl_mem mem) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx || !g || ndev == 0) { set_error("null handle list"); return DBL_E_ARG; }
    if (count && (!u || !v || !codes)) { set_error("null argument"); return DBL_E_ARG; }
    if (mem == DBL_MEM_DEVICE && count) {
        // a batch resident on one GPU: every other GPU reads its slice of the
        // pairs and writes its codes over NVLink (peer access), inside its
        // query kernel -- no staging copies, no collective
        cudaPointerAttributes at{};
        const void *bufs[4] = {u, v, codes, visited};
        int owner = -1;
        for (const void *b : bufs) {
            if (!b) continue;
            if (cudaPointerGetAttributes(&at, b) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
                cudaGetLastError();
                set_error("dbl_query_multi with DBL_MEM_DEVICE needs device buffers");
                return DBL_E_ARG;
            }
            if (owner < 0) owner = at.device;
            if (at.device != owner) { set_error("the batch's buffers live on different devices"); return DBL_E_ARG; }
        }
        for (uint32_t d = 0; d < ndev; ++d) {
            const int dev = g[d]->device;
            if (dev == owner) continue;
            int can = 0;
            DBL_CUDA(cudaDeviceCanAccessPeer(&can, dev, owner));
            if (!can) { set_error("device " + std::to_string(dev) + " has no peer access to the batch's device"); return DBL_E_ARG; }
            DBL_CUDA(cudaSetDevice(dev));
            const cudaError_t e = cudaDeviceEnablePeerAccess(owner, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
        }
    }
    for (uint32_t d = 0; d < ndev; ++d) {
        dbl_status s = check_pair(idx[d], g[d]);
        if (s) return s;
        if (idx[d]->n != idx[0]->n) { set_error("replicas differ in vertex count"); return DBL_E_MISMATCH; }
        for (uint32_t e = 0; e < d; ++e)   // a handle serves one host thread at a time
            if (g[e] == g[d]) { set_error("dbl_query_multi needs distinct graph handles per slice"); return DBL_E_ARG; }
    }
    const uint64_t chunk = ndev ? (count + ndev - 1) / ndev : count;
    std::vector<dbl_status> st(ndev, DBL_OK);
    std::vector<std::string> msg(ndev);
    auto work = [&](uint32_t d) {
        const uint64_t lo = d * chunk < count ? d * chunk : count;
        const uint64_t hi = lo + chunk < count ? lo + chunk : count;
        st[d] = query_impl(idx[d], g[d], u + lo, v + lo, hi - lo, flags, codes + lo, visited ? visited + lo : nullptr,
                           mem, true);
        if (st[d]) msg[d] = g_last_error;
    };
    if (ndev == 1 || count < 2 * (uint64_t)ndev) {
        for (uint32_t d = 0; d < ndev; ++d) work(d);
    } else {
        std::vector<std::thread> th;
        for (uint32_t d = 1; d < ndev; ++d) th.emplace_back(work, d);
        work(0);
        for (auto &t : th) t.join();
    }
    for (uint32_t d = 0; d < ndev; ++d)
        if (st[d]) { set_error("device slice " + std::to_string(d) + ": " + msg[d]); return st[d]; }
    return DBL_OK;
}

// ---------------------------------------------------------------- updates --

static dbl_status count_certified(dbl_graph *g, const dbl_index *idx, const uint64_t *keys, uint64_t count,
                                  uint64_t *out) {
    *out = 0;
    if (!count || !idx->wdl) return DBL_OK;
    DevBuf c;
    dbl_status s = c.ensure(8);
    if (s) return s;
    DBL_CUDA(cudaMemsetAsync(c.p, 0, 8, g->stream));
    certified_kernel<<<grid_for(count), 256, 0, g->stream>>>(idx->rec.as<uint64_t>(), idx->rs, idx->wdl + idx->wbl, idx->wdl, keys,
                                                              count, c.as<unsigned long long>());
    DBL_LAUNCHED();
    unsigned long long h = 0;
    DBL_CUDA(cudaMemcpyAsync(&h, c.p, 8, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    c.release();
    *out = h;
    return DBL_OK;
}

// Same count into a device word (read by the caller after its final sync);
// stream order puts it before the batch's label updates.
static dbl_status count_certified_async(dbl_graph *g, const dbl_index *idx, const uint64_t *keys, uint64_t count,
                                        unsigned long long *dcount, const uint64_t *valid_dev,
                                        const unsigned long long *abort_dev) {
    if (!count || !idx->wdl) return DBL_OK;
    certified_kernel<<<grid_for(count), 256, 0, g->stream>>>(idx->rec.as<uint64_t>(), idx->rs, idx->wdl + idx->wbl, idx->wdl, keys,
                                                              count, dcount, valid_dev, abort_dev);
    DBL_LAUNCHED();
    return DBL_OK;
}

extern "C" dbl_status dbl_insert_edge(dbl_index *idx, dbl_graph *g, uint32_t u, uint32_t v,
                                      dbl_update_stats *stats) {
    dbl_status s = check_pair(idx, g);
    if (s) return s;
    if (u >= g->n || v >= g->n) {
        set_error("vertex " + std::to_string(u >= g->n ? u : v) + " outside [0, " + std::to_string(g->n) + ")");
        return DBL_E_VERTEX_RANGE;
    }
    dbl_update_stats st{};
    bool done = false, dig_ok = false, served = false;
    uint32_t dirs_done = 0;
    // the per-call service runs K9 in its resident CTA (no launch, no sync)
    if ((s = serve_insert(idx, g, u, v, &st, &done, &dirs_done, &dig_ok, &served))) return s;
    if (served && done) {
        if (stats) *stats = st;
        return DBL_OK;
    }
    ServeBlock no_service_;   // K9 launch and the batch fixpoint: no per-call service runs during them
    if (!served) {
        DBL_CUDA(cudaSetDevice(g->device));
        set_stream(g->stream);
        // the fast path ORs each written label delta's digest bits into the
        // digest (digest bits are ORs of label bits), the fallback refreshes
        // the changed vertices, so a current digest stays current
        dig_ok = idx->digest_version == idx->version;
        ++idx->version;
        // one launch + one sync: pre-check, add_edge into the pending log,
        // both propagations (insert_one.cu)
        if ((s = insert_edge_fast(idx, g, u, v, &st, &done, &dirs_done, dig_ok))) return s;
        if (done && dig_ok) idx->digest_version = idx->version;
    }
    if (done) {
        if (stats) *stats = st;
        return DBL_OK;
    }
    DBL_CUDA(cudaSetDevice(g->device));
    set_stream(g->stream);
    // a cone outgrew the single-CTA tables (no label was written; the edge is
    // in the graph): fold the log into the delta adjacency and run the batch
    // fixpoint from this edge's seeds
    if ((s = graph_flush_pending(g))) return s;
    const uint64_t key = ((uint64_t)u << 32) | v;
    DevBuf kb;
    if ((s = kb.ensure(16))) return s;
    DBL_CUDA(cudaMemcpyAsync(kb.p, &key, 8, cudaMemcpyHostToDevice, g->stream));
    uint32_t changed[2], seedc[2], levels = 0;
    s = run_insert(g, idx, kb.as<uint64_t>(), 1, true, changed, seedc, &levels);
    kb.release();
    if (s || (s = digest_after_insert(idx, g, dig_ok))) return s;
    // _propagate_union dequeues the seed plus every changed non-seed vertex;
    // a direction the fast path already finished (its labels are final, so
    // the fixpoint changes nothing there) keeps the fast path's counts
    for (int d = 0; d < 2; ++d) {
        if ((dirs_done >> d) & 1u) continue;
        st.visited += 1 + changed[d] - seedc[d];
        st.labels_changed += changed[d];
    }
    if (stats) *stats = st;
    return DBL_OK;
}

extern "C" dbl_status dbl_insert_edges(dbl_index *idx, dbl_graph *g, const uint32_t *u, const uint32_t *v,
                                       uint64_t count, dbl_mem mem, dbl_batch_stats *stats) {
    ServeBlock no_service_;   // no per-call service runs during this call
    dbl_status s = check_pair(idx, g);
    if (s) return s;
    dbl_batch_stats st{};
    st.requested = count;
    if (!count) { if (stats) *stats = st; return DBL_OK; }
    if (!u || !v) { set_error("null argument"); return DBL_E_ARG; }
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    const bool dig_ok = idx->digest_version == idx->version;   // kept current by the change bitmaps
    ++idx->version;
    trace("insert: enter", g->stream);
    // the batch's workspaces stay with the graph (grow-only): no pool round
    // trips per batch
    DevBuf &in = g->ins_in, &keys = g->ins_keys, &alt = g->ins_alt, &newk = g->ins_newk, &err = g->ins_err;
    auto cleanup = [&]() {};
    if ((s = keys.ensure(count * 8)) || (s = alt.ensure(count * 8)) || (s = newk.ensure(count * 8)) ||
        (s = err.ensure(32))) { cleanup(); return s; }
    trace("insert: workspaces", g->stream);
    const uint32_t *du = u, *dv = v;
    if (mem == DBL_MEM_HOST) {
        if ((s = in.ensure(count * 8))) { cleanup(); return s; }
        DBL_CUDA(cudaMemcpyAsync(in.p, u, count * 4, cudaMemcpyHostToDevice, g->stream));
        DBL_CUDA(cudaMemcpyAsync(in.as<uint32_t>() + count, v, count * 4, cudaMemcpyHostToDevice, g->stream));
        du = in.as<uint32_t>();
        dv = du + count;
    } else if ((s = order_after_caller(g))) {
        cleanup();
        return s;
    }
    // st4: [0] vertex-range flag, [1] certified count, [2] new-edge count,
    // [3] unique count.  The whole batch is enqueued without a host round
    // trip: counts stay on the device (the batch size bounds every launch)
    // and a range error turns the batch into a no-op (no new edges), reported
    // after the single readback -- the graph and labels are left as they were.
    trace("insert: ordered", g->stream);
    unsigned long long *st4 = err.as<unsigned long long>();
    DBL_CUDA(cudaMemsetAsync(st4, 0, 32, g->stream));
    trace("insert: memset", g->stream);
    // the batch is sorted on (u << b | v), b = vertex-id bits: 2b radix bits
    // instead of 32 + b (5 onesweep passes instead of 7 at n = 2^20)
    const uint32_t shift = (uint32_t)key_end_bit(g->n) - 32;
    pack_pairs_kernel<<<grid_for(count), 256, 0, g->stream>>>(du, dv, count, g->n, keys.as<uint64_t>(), st4, shift);
    DBL_LAUNCHED();
    uint64_t *sorted = nullptr;
    trace("insert: packed", g->stream);
    if ((s = sort_keys_replay(g, keys.as<uint64_t>(), alt.as<uint64_t>(), count, (int)(2 * shift), &sorted))) {
        cleanup();
        return s;
    }
    trace("insert: sorted", g->stream);
    // unique (into the other buffer); its count goes to st4[3]
    uint64_t *uniq = sorted == keys.as<uint64_t>() ? alt.as<uint64_t>() : keys.as<uint64_t>();
    const uint64_t *dnu = reinterpret_cast<const uint64_t *>(st4 + 3);
    {
        if ((s = cub_cached(g, CUB_UNIQUE, count, 0, [&](void *t, size_t &bytes) {
                 return cub::DeviceSelect::Unique(t, bytes, sorted, uniq, (uint64_t *)(st4 + 3), (int64_t)count,
                                                  g->stream);
             }))) {
            cleanup();
            return s;
        }
        widen_keys_kernel<<<grid_for(count), 256, 0, g->stream>>>(uniq, count, shift, dnu);
        DBL_LAUNCHED();
    }
    trace("insert: sort+unique", g->stream);
    if ((s = count_certified_async(g, idx, uniq, count, st4 + 1, dnu, st4))) { cleanup(); return s; }
    uint64_t nnew = 0;
    bool cert_read = false;
    const uint64_t *dnew = nullptr;
    if ((s = graph_filter_new(g, uniq, count, newk.as<uint64_t>(), &nnew, &dnew, dnu, st4))) { cleanup(); return s; }
    trace("insert: certified+filter", g->stream);
    bool range_error = false;
    {
        const uint64_t nd = g->m_delta;
        DBL_CUDA(cudaMemcpyAsync(st4 + 2, dnew, 8, cudaMemcpyDeviceToDevice, g->stream));
        if ((s = graph_insert_delta(g, newk.as<uint64_t>(), count, dnew))) { cleanup(); return s; }
        trace("insert: delta merge", g->stream);
        uint32_t changed[2], seedc[2], levels = 0;
        unsigned long long hx[4] = {0, 0, 0, 0};
        if ((s = run_insert(g, idx, newk.as<uint64_t>(), count, true, changed, seedc, &levels, st4, hx, dnew))) {
            cleanup();
            return s;
        }
        range_error = hx[0] != 0;
        if (!range_error && (s = digest_after_insert(idx, g, dig_ok))) { cleanup(); return s; }
        st.certified = hx[1];
        nnew = hx[2];
        cert_read = true;
        g->m_delta = nd + nnew;   // settle the upper bound used while enqueueing
        st.inserted = nnew;
        st.labels_changed = (uint64_t)changed[0] + changed[1];
        st.levels = levels;
        st.fix_items = g->last_insert.fix_items;
        st.fix_edges = g->last_insert.fix_edges;
        if (!range_error && g->m_delta * 4 > g->m_base + 1024) {
            if ((s = graph_compact(g))) { cleanup(); return s; }
            st.delta_merged = 1;
        }
    }
    trace("insert: done", g->stream);
    if (range_error) { cleanup(); set_error("insert vertex outside [0, n)"); return DBL_E_VERTEX_RANGE; }
    if (!cert_read) {
        unsigned long long hcert = 0;
        DBL_CUDA(cudaMemcpyAsync(&hcert, err.p, 8, cudaMemcpyDeviceToHost, g->stream));
        DBL_CUDA(cudaStreamSynchronize(g->stream));
        st.certified = hcert;
    }
    cleanup();
    if (stats) *stats = st;
    return DBL_OK;
}

extern "C" dbl_status dbl_work_model(const dbl_index *idx, const dbl_graph *gc, uint64_t *V, uint64_t *E,
                                     uint32_t *levels) {
    ServeBlock no_service_;   // no per-call service runs during this call
    dbl_status s = check_pair(idx, gc);
    if (s) return s;
    if (!V || !E || !levels) { set_error("null argument"); return DBL_E_ARG; }
    dbl_graph *g = const_cast<dbl_graph *>(gc);
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    return work_model(idx, g, V, E, levels);
}

// -------------------------------------------------- multi-GPU word shards --

__global__ void pack_words_kernel(const uint64_t *__restrict__ rec, uint32_t rs, uint32_t n,
                                  const uint32_t *__restrict__ words, uint32_t nw, uint64_t *__restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)n * nw;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(i / n), v = (uint32_t)(i % n);
        out[i] = rec[(size_t)v * rs + words[j]];
    }
}

__global__ void unpack_words_kernel(uint64_t *__restrict__ rec, uint32_t rs, uint32_t n,
                                    const uint32_t *__restrict__ words, uint32_t nw, const uint64_t *__restrict__ in) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)n * nw;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(i / n), v = (uint32_t)(i % n);
        rec[(size_t)v * rs + words[j]] = in[i];
    }
}

// Pack record words `words` (host list) of every vertex into a word-major
// slab (nw x n u64, device memory) -- the unit of the NCCL allgather.
extern "C" dbl_status dbl_index_pack_words(const dbl_index *idx, const uint32_t *words, uint32_t nw,
                                           uint64_t *dev_slab, void *stream) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx || (nw && (!words || !dev_slab))) { set_error("null argument"); return DBL_E_ARG; }
    if (!nw || !idx->n) return DBL_OK;
    DBL_CUDA(cudaSetDevice(idx->device));
    set_stream(nullptr);
    DevBuf w;
    dbl_status s = w.ensure(nw * 4);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    set_stream(st);
    DBL_CUDA(cudaMemcpyAsync(w.p, words, nw * 4, cudaMemcpyHostToDevice, st));
    pack_words_kernel<<<grid_for((uint64_t)idx->n * nw), 256, 0, st>>>(idx->rec.as<uint64_t>(), idx->rs, idx->n,
                                                                       w.as<uint32_t>(), nw, dev_slab);
    DBL_LAUNCHED();
    DBL_CUDA(cudaStreamSynchronize(st));
    w.release();
    return DBL_OK;
}

// Inverse of dbl_index_pack_words: scatter a slab (K5 record interleave).
extern "C" dbl_status dbl_index_unpack_words(dbl_index *idx, const uint32_t *words, uint32_t nw,
                                             const uint64_t *dev_slab, void *stream) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx || (nw && (!words || !dev_slab))) { set_error("null argument"); return DBL_E_ARG; }
    if (!nw || !idx->n) return DBL_OK;
    DBL_CUDA(cudaSetDevice(idx->device));
    set_stream(nullptr);
    DevBuf w;
    dbl_status s = w.ensure(nw * 4);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    set_stream(st);
    ++idx->version;
    DBL_CUDA(cudaMemcpyAsync(w.p, words, nw * 4, cudaMemcpyHostToDevice, st));
    unpack_words_kernel<<<grid_for((uint64_t)idx->n * nw), 256, 0, st>>>(idx->rec.as<uint64_t>(), idx->rs, idx->n,
                                                                         w.as<uint32_t>(), nw, dev_slab);
    DBL_LAUNCHED();
    DBL_CUDA(cudaStreamSynchronize(st));
    w.release();
    return DBL_OK;
}

// ------------------------------------------------------- graph-only edges --

// DynamicGraph.add_edge for a batch without label maintenance (graph.py:56-66):
// out_new (host, optional) receives 1 for each pair that was absent before the
// call and not repeated earlier in the batch.
extern "C" dbl_status dbl_graph_add_edges(dbl_graph *g, const uint32_t *u, const uint32_t *v, uint64_t count,
                                          uint64_t *out_inserted) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!g || (count && (!u || !v))) { set_error("null argument"); return DBL_E_ARG; }
    if (out_inserted) *out_inserted = 0;
    if (!count) return DBL_OK;
    DBL_CUDA(cudaSetDevice(g->device));
    if (dbl_status fs = graph_flush_pending(const_cast<dbl_graph *>(g))) return fs;
    set_stream(g->stream);
    DevBuf in, keys, alt, newk, err;
    auto cleanup = [&]() { in.release(); keys.release(); alt.release(); newk.release(); err.release(); };
    dbl_status s;
    if ((s = in.ensure(count * 8)) || (s = keys.ensure(count * 8)) || (s = alt.ensure(count * 8)) ||
        (s = newk.ensure(count * 8)) || (s = err.ensure(16))) { cleanup(); return s; }
    DBL_CUDA(cudaMemcpyAsync(in.p, u, count * 4, cudaMemcpyHostToDevice, g->stream));
    DBL_CUDA(cudaMemcpyAsync(in.as<uint32_t>() + count, v, count * 4, cudaMemcpyHostToDevice, g->stream));
    DBL_CUDA(cudaMemsetAsync(err.p, 0, 16, g->stream));
    pack_pairs_kernel<<<grid_for(count), 256, 0, g->stream>>>(in.as<uint32_t>(), in.as<uint32_t>() + count, count,
                                                              g->n, keys.as<uint64_t>(), err.as<unsigned long long>());
    DBL_LAUNCHED();
    unsigned long long herr = 0;
    DBL_CUDA(cudaMemcpyAsync(&herr, err.p, 8, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    if (herr) { cleanup(); set_error("edge endpoint outside [0, n)"); return DBL_E_VERTEX_RANGE; }
    uint64_t *sorted = nullptr;
    if ((s = sort_keys(g, keys.as<uint64_t>(), alt.as<uint64_t>(), count, key_end_bit(g->n), &sorted))) {
        cleanup();
        return s;
    }
    uint64_t *uniq = sorted == keys.as<uint64_t>() ? alt.as<uint64_t>() : keys.as<uint64_t>();
    size_t tmp = 0;
    uint64_t *dn = err.as<uint64_t>() + 1;
    DBL_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, sorted, uniq, dn, (int64_t)count, g->stream));
    if ((s = g->cub_tmp.ensure(tmp))) { cleanup(); return s; }
    DBL_CUDA(cub::DeviceSelect::Unique(g->cub_tmp.p, tmp, sorted, uniq, dn, (int64_t)count, g->stream));
    DBL_LAUNCHED();
    uint64_t nu = 0, nnew = 0;
    DBL_CUDA(cudaMemcpyAsync(&nu, dn, 8, cudaMemcpyDeviceToHost, g->stream));
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    if ((s = graph_filter_new(g, uniq, nu, newk.as<uint64_t>(), &nnew))) { cleanup(); return s; }
    if (nnew && (s = graph_insert_delta(g, newk.as<uint64_t>(), nnew))) { cleanup(); return s; }
    if (nnew && g->m_delta * 4 > g->m_base + 1024) s = graph_compact(g);
    cleanup();
    if (s) return s;
    if (out_inserted) *out_inserted = nnew;
    DBL_CUDA(cudaStreamSynchronize(g->stream));
    return DBL_OK;
}

// --------------------------------------------------------- label helpers --

__global__ void label_tests_kernel(const uint64_t *__restrict__ rec, uint32_t wdl, uint32_t wbl, uint32_t n,
                                   const uint32_t *__restrict__ x, const uint32_t *__restrict__ y, uint64_t count,
                                   uint8_t *__restrict__ dl, uint8_t *__restrict__ bl, unsigned long long *err) {
    const uint32_t H = wdl + wbl, rs = rec_stride(H);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = x[i], b = y[i];
        if (a >= n || b >= n) { atomicOr(err, 1ull); continue; }
        const uint64_t *ra = rec + (size_t)a * rs, *rb = rec + (size_t)b * rs;
        uint64_t d = 0, c = 0;
        for (uint32_t k = 0; k < wdl; ++k) d |= ra[H + k] & rb[k];
        for (uint32_t k = 0; k < wbl; ++k) c |= (ra[wdl + k] & ~rb[wdl + k]) | (rb[H + wdl + k] & ~ra[H + wdl + k]);
        dl[i] = d != 0;
        bl[i] = c == 0;
    }
}

// dl_intersec (labels.py:315-319) and bl_contain (labels.py:322-327) for a
// batch of (x, y) pairs, host in/out.
extern "C" dbl_status dbl_label_tests(const dbl_index *idx, const uint32_t *x, const uint32_t *y, uint64_t count,
                                      uint8_t *out_dl_intersec, uint8_t *out_bl_contain) {
    ServeBlock no_service_;   // no per-call service runs during this call
    if (!idx || (count && (!x || !y || !out_dl_intersec || !out_bl_contain))) {
        set_error("null argument");
        return DBL_E_ARG;
    }
    if (!count) return DBL_OK;
    DBL_CUDA(cudaSetDevice(idx->device));
    set_stream(nullptr);
    DevBuf b;
    dbl_status s = b.ensure(count * 10 + 16);
    if (s) return s;
    uint32_t *dx = b.as<uint32_t>(), *dy = dx + count;
    uint8_t *ddl = reinterpret_cast<uint8_t *>(dy + count), *dbl = ddl + count;
    unsigned long long *derr = reinterpret_cast<unsigned long long *>(b.as<char>() + ((count * 10 + 7) & ~7ull));
    cudaMemcpy(dx, x, count * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, y, count * 4, cudaMemcpyHostToDevice);
    cudaMemset(derr, 0, 8);
    label_tests_kernel<<<grid_for(count), 256>>>(idx->rec.as<uint64_t>(), idx->wdl, idx->wbl, idx->n, dx, dy, count,
                                                 ddl, dbl, derr);
    DBL_LAUNCHED();
    unsigned long long herr = 0;
    cudaMemcpy(out_dl_intersec, ddl, count, cudaMemcpyDeviceToHost);
    cudaMemcpy(out_bl_contain, dbl, count, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaMemcpy(&herr, derr, 8, cudaMemcpyDeviceToHost);
    b.release();
    if (e != cudaSuccess) return cuda_fail(e, "label_tests");
    if (herr) { set_error("vertex outside [0, n)"); return DBL_E_VERTEX_RANGE; }
    return DBL_OK;
}
