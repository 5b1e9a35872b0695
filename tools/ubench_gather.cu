// Random-line gather microbenchmark: the memory pattern of the query label
// check (two random records per query).  Each thread reads `bytes` (32..128)
// at a random line-aligned offset of a `size` buffer, for buffer sizes from
// below L2 to far above it, and reports GB/s of bytes requested and of whole
// 128-byte lines touched.  Tells how much of the HBM copy bandwidth a random
// gather can reach on this part, and whether the footprint (TLB reach) costs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_gather tools/ubench_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

template <int B>
__global__ void __launch_bounds__(256) gather(const uint64_t *__restrict__ buf, uint64_t lines, uint64_t n,
                                              uint64_t seed, uint64_t *__restrict__ out) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t *p = buf + (mix(i ^ seed) % lines) * 16;
#pragma unroll
        for (int k = 0; k < B / 8; k += 4) {
            uint64_t a, b, c, d;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                         : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p + k));
            acc ^= a ^ b ^ c ^ d;
        }
    }
    if (acc == 0x1234567) out[0] = acc;
}

// 4 lanes per line: lane j of a quad reads bytes [32j, 32j + 32) of the
// quad's line, so a warp instruction is one request per line (4 sectors)
__global__ void __launch_bounds__(256) gather_quad(const uint64_t *__restrict__ buf, uint64_t lines, uint64_t n,
                                                   uint64_t seed, uint64_t *__restrict__ out) {
    uint64_t acc = 0;
    const int q = threadIdx.x & 3;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 4 * n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t *p = buf + (mix((i >> 2) ^ seed) % lines) * 16 + q * 4;
        uint64_t a, b, c, d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        acc ^= a ^ b ^ c ^ d;
    }
    if (acc == 0x1234567) out[0] = acc;
}

int main() {
    const size_t maxb = 32ull << 30;
    uint64_t *buf, *out;
    if (cudaMalloc(&buf, maxb) != cudaSuccess) { std::printf("alloc failed\n"); return 1; }
    cudaMalloc(&out, 64);
    cudaMemset(buf, 1, maxb);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint64_t n = 64ull << 20;   // accesses per launch
    for (size_t sz : {64ull << 20, 256ull << 20, 1ull << 30, 4ull << 30, 8ull << 30, 16ull << 30, 32ull << 30}) {
        const uint64_t lines = sz / 128;
        {
            float best = 1e9f;
            for (int r = 0; r < 4; ++r) {
                cudaEventRecord(e0);
                gather_quad<<<sms * 8, 256>>>(buf, lines, n, r * 77 + 1, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r && ms < best) best = ms;
            }
            std::printf("size %6.2f GB  quad-128  %.3f ms  %.0f GB/s  %.2f G lines/s\n", sz / 1073741824.0, best,
                        n * 128.0 / best / 1e6, n / best / 1e6);
        }
        for (int bytes : {32, 128}) {
            for (int ctas : {8}) {   // resident 256-thread CTAs per SM
                const int grid = sms * ctas;
                float best = 1e9f;
                for (int r = 0; r < 4; ++r) {
                    cudaEventRecord(e0);
                    if (bytes == 32) gather<32><<<grid, 256>>>(buf, lines, n, r * 77 + 1, out);
                    else if (bytes == 64) gather<64><<<grid, 256>>>(buf, lines, n, r * 77 + 1, out);
                    else gather<128><<<grid, 256>>>(buf, lines, n, r * 77 + 1, out);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (r && ms < best) best = ms;
                }
                std::printf("size %6.2f GB  bytes %3d  ctas/sm %d  %.3f ms  req %.0f GB/s  lines %.0f GB/s  %.2f G acc/s\n",
                            sz / 1073741824.0, bytes, ctas, best, n * bytes / best / 1e6,
                            n * 128.0 / best / 1e6, n / best / 1e6);
            }
        }
    }
    return 0;
}
