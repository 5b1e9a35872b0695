// Per-call overhead of the synchronous query API against the CUDA floor on
// this box: an empty kernel + stream sync, an empty kernel + 32-byte D2H copy
// + sync, and dbl_query / dbl_query_async + dbl_sync on a 1-query batch.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o tools/ubench_api \
//        tools/ubench_api.cu -Lpaper_2101_09441_b200/_lib -ldbl_b200 -Xlinker -rpath=$PWD/paper_2101_09441_b200/_lib
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "dbl_b200.h"

__global__ void empty_kernel() {}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Mailbox ping-pong over pinned host memory: one thread polls mb[0] and
// echoes each new value into resp[0] (the floor of a persistent "query
// server" kernel).  Exits after `iters` requests or 2 s, whichever first.
__global__ void pingpong(volatile uint32_t *mb, volatile uint32_t *resp, int iters) {
    if (threadIdx.x) return;
    const unsigned long long t0 = gtime();
    uint32_t last = 0;
    for (int i = 0; i < iters; ++i) {
        uint32_t s;
        do {
            s = mb[0];
            if (gtime() - t0 > 2000000000ull) return;
        } while (s == last);
        last = s;
        resp[0] = s;
        __threadfence_system();
    }
}

template <typename F>
static double med_us(F f, int n = 400) {
    std::vector<double> t;
    for (int i = 0; i < n; ++i) {
        auto a = std::chrono::steady_clock::now();
        f();
        auto b = std::chrono::steady_clock::now();
        if (i >= 20) t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    const uint32_t n = 1 << 16;
    std::vector<uint32_t> src, dst;
    for (uint32_t i = 0; i + 1 < n; ++i) { src.push_back(i); dst.push_back((i * 7 + 1) % n); }
    dbl_graph *g = nullptr;
    dbl_index *idx = nullptr;
    if (dbl_graph_create(n, src.data(), dst.data(), src.size(), DBL_MEM_HOST, 0, &g)) { std::printf("graph failed\n"); return 1; }
    dbl_config cfg{64, 64, 0, 0, 0};
    if (dbl_index_build(g, &cfg, nullptr, nullptr, nullptr, nullptr, nullptr, 0, &idx)) { std::printf("build failed\n"); return 1; }
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    uint32_t *du, *dv, *hres;
    uint8_t *dc;
    cudaMalloc(&du, 64); cudaMalloc(&dv, 64); cudaMalloc(&dc, 64);
    cudaMemset(du, 0, 64); cudaMemset(dv, 0, 64);
    cudaHostAlloc(&hres, 64, 0);
    uint32_t hu = 1, hv = 2;
    uint8_t hc = 0;
    std::printf("empty kernel + sync:              %6.1f us\n", med_us([&] { empty_kernel<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }));
    std::printf("empty kernel + 32 B D2H + sync:   %6.1f us\n", med_us([&] {
        empty_kernel<<<1, 32, 0, s>>>(); cudaMemcpyAsync(hres, du, 32, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }));
    std::printf("dbl_query, device, 1 query:       %6.1f us\n", med_us([&] { dbl_query(idx, g, du, dv, 1, 0x3f, dc, nullptr, DBL_MEM_DEVICE); }));
    std::printf("dbl_query, host (pageable), 1 q:  %6.1f us\n", med_us([&] { dbl_query(idx, g, &hu, &hv, 1, 0x3f, &hc, nullptr, DBL_MEM_HOST); }));
    std::printf("dbl_query_async + dbl_sync, 1 q:  %6.1f us\n", med_us([&] { dbl_query_async(idx, g, du, dv, 1, 0x3f, dc, nullptr); dbl_sync(g); }));
    {
        uint32_t *mb, *resp;
        cudaHostAlloc(&mb, 64, cudaHostAllocMapped);
        cudaHostAlloc(&resp, 64, cudaHostAllocMapped);
        mb[0] = 0;
        resp[0] = 0;
        cudaStream_t s2;
        cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
        const int iters = 2000;
        pingpong<<<1, 32, 0, s2>>>(mb, resp, iters);
        std::vector<double> t;
        bool ok = true;
        for (int i = 1; i <= iters && ok; ++i) {
            auto a = std::chrono::steady_clock::now();
            *(volatile uint32_t *)mb = (uint32_t)i;
            while (*(volatile uint32_t *)resp != (uint32_t)i) {
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count() > 1.0) { ok = false; break; }
            }
            auto b = std::chrono::steady_clock::now();
            if (i > 20) t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
        }
        cudaStreamSynchronize(s2);
        std::sort(t.begin(), t.end());
        if (ok && !t.empty())
            std::printf("mailbox ping-pong (pinned):       %6.2f us (p10 %.2f, p90 %.2f)\n", t[t.size() / 2],
                        t[t.size() / 10], t[t.size() * 9 / 10]);
        else
            std::printf("mailbox ping-pong: timed out\n");
    }
    uint32_t *pu, *pv;
    uint8_t *pc;
    const size_t Q = 1 << 20;
    cudaHostAlloc(&pu, Q * 4, 0); cudaHostAlloc(&pv, Q * 4, 0); cudaHostAlloc(&pc, Q, 0);
    for (size_t i = 0; i < Q; ++i) { pu[i] = (uint32_t)((i * 2654435761u) % n); pv[i] = (uint32_t)((i * 40503u + 7) % n); }
    cudaPointerAttributes at{};
    std::printf("cudaPointerGetAttributes (pinned):%6.2f us\n", med_us([&] { cudaPointerGetAttributes(&at, pu); }));
    std::printf("dbl_query, host pinned, 1 query:  %6.1f us\n", med_us([&] { dbl_query(idx, g, pu, pv, 1, 0x3f, pc, nullptr, DBL_MEM_HOST); }));
    std::printf("dbl_query, host pinned, 2^20 q:   %6.1f us\n", med_us([&] { dbl_query(idx, g, pu, pv, Q, 0x3f, pc, nullptr, DBL_MEM_HOST); }, 60));
    return 0;
}
