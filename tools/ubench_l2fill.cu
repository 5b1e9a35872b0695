// Cold-L2 random gather over a table smaller than L2 (the cfg2 query shape:
// 2M random 32-byte records of a 32 MB table right after an L2 flush), with
// and without filling L2 first.  Variants: no fill; bulk L2 prefetch
// (cp.async.bulk.prefetch.L2) in the same kernel; per-line prefetch.global.L2
// in the same kernel; a coalesced read pass in the same kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_l2fill tools/ubench_l2fill.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

// mode 0: none, 1: bulk prefetch, 2: prefetch.global.L2 per line, 3: coalesced loads
__global__ void __launch_bounds__(256) gather(const uint64_t *__restrict__ tab, uint64_t recs, uint64_t n, int mode,
                                              uint64_t seed, uint64_t *__restrict__ out) {
    const uint64_t bytes = recs * 32;
    const uint64_t slice = ((bytes + gridDim.x - 1) / gridDim.x + 127) & ~127ull;
    const uint64_t b0 = blockIdx.x * slice;
    const char *base = reinterpret_cast<const char *>(tab);
    uint64_t acc = 0;
    if (b0 < bytes) {
        const uint64_t len = min(slice, bytes - b0);
        if (mode == 1) {
            for (uint64_t off = threadIdx.x * 4096ull; off < len; off += blockDim.x * 4096ull) {
                const uint32_t sz = (uint32_t)min((uint64_t)4096, len - off);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + b0 + off), "r"(sz) : "memory");
            }
        } else if (mode == 2) {
            for (uint64_t off = threadIdx.x * 128ull; off < len; off += blockDim.x * 128ull)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(base + b0 + off));
        } else if (mode == 3) {
            for (uint64_t off = threadIdx.x * 32ull; off < len; off += blockDim.x * 32ull) {
                uint64_t a, b, c, d;
                asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                             : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(base + b0 + off));
                acc ^= a;
            }
        }
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t *p = tab + (mix(i ^ seed) % recs) * 4;
        uint64_t a, b, c, d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        acc ^= a ^ b ^ c ^ d;
    }
    if (acc == 0x1234567) out[0] = acc;
}

__global__ void flush_kernel(uint64_t *f, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        f[i] += 1;
}

int main() {
    uint64_t *tab, *out, *fl;
    const uint64_t flw = (512ull << 20) / 8;
    cudaMalloc(&tab, 256ull << 20);
    cudaMalloc(&out, 64);
    cudaMalloc(&fl, flw * 8);
    cudaMemset(tab, 1, 256ull << 20);
    cudaMemset(fl, 0, flw * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (uint64_t mb : {8ull, 32ull, 64ull}) {
        const uint64_t recs = (mb << 20) / 32;
        for (uint64_t n : {1ull << 20, 2ull << 20, 4ull << 20}) {
            for (int mode = 0; mode < 4; ++mode) {
                float sum = 0;
                const int reps = 6;
                for (int r = 0; r < reps; ++r) {
                    flush_kernel<<<sms * 8, 256>>>(fl, flw);
                    cudaEventRecord(e0);
                    gather<<<sms * 8, 256>>>(tab, recs, n, mode, r * 131 + 7, out);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (r) sum += ms;
                }
                std::printf("table %3llu MB  accesses %5.2f M  mode %d  %.2f us\n", (unsigned long long)mb, n / 1048576.0,
                            mode, 1000.0f * sum / (reps - 1));
            }
        }
    }
    return 0;
}
