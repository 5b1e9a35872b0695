// HBM write ceiling for the build's record write-out (reach_kernel's apply
// phase writes n records of 128 B: 8.6 GB at cfg5).  Compares cudaMemset,
// plain streaming stores of 16 and 32 bytes per lane, and the apply
// pattern (a bitmap word + a flag byte per vertex read, then the 32 records
// of a 32-vertex block written with 512-byte warp stores), at several grid
// sizes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_write tools/ubench_write.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void st16(uint4 *p, size_t n16) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    for (; i < n16; i += s) p[i] = make_uint4(i, 0, 0, 0);
}

__global__ void st32(uint64_t *p, size_t n32) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    for (; i < n32; i += s) {
        uint64_t *q = p + 4 * i;
        asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(q), "l"((uint64_t)i), "l"(0ull), "l"(0ull),
                     "l"(0ull) : "memory");
    }
}

// 32-byte stores covering only the first 3 sectors of every 128-byte line
// (records of 80 bytes at a 128-byte stride with the pad sector skipped)
__global__ void st32_skip(uint64_t *p, size_t n32) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    for (; i < n32; i += s) {
        if ((i & 3) == 3) continue;
        uint64_t *q = p + 4 * i;
        asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(q), "l"((uint64_t)i), "l"(0ull), "l"(0ull),
                     "l"(0ull) : "memory");
    }
}

// the apply pattern: a warp per 32-vertex block; read vis word + 32 flag
// bytes, then 8 x 512-byte stores of the block's 32 x 128-byte records
template <bool CS>
__global__ void apply_like(uint64_t *rec, const uint32_t *vis, const uint8_t *flags, uint32_t n, uint64_t acc) {
    const int lane = threadIdx.x & 31;
    const uint64_t nblk = (n + 31) / 32, gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5,
                   nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t blk = gw; blk < nblk; blk += nw) {
        const uint32_t fb = vis[blk];
        const uint8_t f = flags[blk * 32 + lane];
        uint64_t *base = rec + blk * 32 * 16;
#pragma unroll
        for (uint32_t t = 0; t < 16 * 32; t += 64) {
            const uint32_t wi = t + 2 * lane, r = wi / 16;
            const uint32_t sf = __shfl_sync(0xffffffffu, (uint32_t)f, r);
            ulonglong2 v;
            v.x = ((fb >> r) & 1u) ? acc : sf;
            v.y = 0;
            if (CS)
                __stcs(reinterpret_cast<ulonglong2 *>(base + wi), v);
            else
                *reinterpret_cast<ulonglong2 *>(base + wi) = v;
        }
    }
}

int main() {
    const size_t bytes = 8ull << 30;
    const uint32_t n = (uint32_t)(bytes / 128);
    uint64_t *rec; uint32_t *vis; uint8_t *flags; char *src;
    CK(cudaMalloc(&rec, bytes));
    CK(cudaMalloc(&src, 4ull << 30));
    CK(cudaMalloc(&vis, n / 8 + 64));
    CK(cudaMalloc(&flags, n + 64));
    CK(cudaMemset(vis, 0x55, n / 8 + 64));
    CK(cudaMemset(flags, 1, n + 64));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto rep = [&](const char *name, double gb, auto fn) {
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r && ms < best) best = ms;
        }
        printf("%-36s %8.3f ms  %7.0f GB/s\n", name, best, gb / best * 1e3);
    };
    const double gb = bytes / 1e9;
    rep("cudaMemset 8 GiB", gb, [&] { cudaMemsetAsync(rec, 0, bytes); });
    rep("cudaMemcpy D2D 4 GiB (r+w)", 2 * 4.294967296, [&] { cudaMemcpyAsync(rec, src, 4ull << 30, cudaMemcpyDeviceToDevice); });
    for (int per : {4, 8, 16}) {
        char name[64];
        snprintf(name, sizeof name, "st16 grid %d x 256", sms * per);
        rep(name, gb, [&] { st16<<<sms * per, 256>>>((uint4 *)rec, bytes / 16); });
        snprintf(name, sizeof name, "st32 grid %d x 256", sms * per);
        rep(name, gb, [&] { st32<<<sms * per, 256>>>(rec, bytes / 32); });
        snprintf(name, sizeof name, "st32 3-of-4 sectors grid %d x 256", sms * per);
        rep(name, gb, [&] { st32_skip<<<sms * per, 256>>>(rec, bytes / 32); });
        snprintf(name, sizeof name, "apply-like grid %d x 256", sms * per);
        rep(name, gb, [&] { apply_like<false><<<sms * per, 256>>>(rec, vis, flags, n, 7); });
        snprintf(name, sizeof name, "apply-like .cs grid %d x 256", sms * per);
        rep(name, gb, [&] { apply_like<true><<<sms * per, 256>>>(rec, vis, flags, n, 7); });
    }
    CK(cudaGetLastError());
    return 0;
}
