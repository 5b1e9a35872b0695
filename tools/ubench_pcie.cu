// Host->device transfer rates for the end-to-end query path: 8 MB of pinned
// (u, v) pairs and 1 MB of codes back.  (a) copy-engine cudaMemcpyAsync, one
// transfer and in chunks on two streams; (b) kernels reading the pinned
// buffer directly (zero-copy) with 4-, 8- and 16-byte loads per thread;
// (c) zero-copy 1 MB device->host writes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_pcie tools/ubench_pcie.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename T>
__global__ void zc_read(const T *__restrict__ h, size_t n, unsigned long long *out) {
    unsigned long long acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const T x = h[i];
        acc += reinterpret_cast<const uint32_t *>(&x)[0];
    }
    if (acc == 0x12345) *out = acc;
}

__global__ void zc_write(uint8_t *h, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 4; i += (size_t)gridDim.x * blockDim.x)
        reinterpret_cast<uint32_t *>(h)[i] = (uint32_t)i;
}

int main() {
    const size_t bytes = 8u << 20, obytes = 1u << 20;
    void *h, *ho, *d;
    unsigned long long *out;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&ho, obytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    cudaMalloc(&out, 8);
    void *hd, *hod;
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaHostGetDevicePointer(&hod, ho, 0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t s0, s1;
    cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto fn, double mb) {
        float best = 1e9f, sum = 0;
        for (int r = 0; r < 8; ++r) {
            cudaEventRecord(e0, s0);
            fn();
            cudaEventRecord(e1, s0);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r) { sum += ms; if (ms < best) best = ms; }
        }
        std::printf("%-40s best %7.1f us  mean %7.1f us  %6.1f GB/s (best)\n", name, best * 1e3, sum / 7 * 1e3,
                    mb / best);
    };
    timeit("memcpy H2D 8 MB", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s0); }, bytes / 1e6);
    for (int ch : {2, 4, 8}) {
        char name[64];
        std::snprintf(name, sizeof name, "memcpy H2D 8 MB in %d chunks, 2 streams", ch);
        timeit(name, [&] {
            cudaEvent_t es;
            cudaEventCreateWithFlags(&es, cudaEventDisableTiming);
            cudaEventRecord(es, s0);   // s1 starts after the timing event on s0
            cudaStreamWaitEvent(s1, es, 0);
            cudaEventDestroy(es);
            for (int i = 0; i < ch; ++i) {
                cudaStream_t st = (i & 1) ? s1 : s0;
                cudaMemcpyAsync((char *)d + i * (bytes / ch), (char *)h + i * (bytes / ch), bytes / ch,
                                cudaMemcpyHostToDevice, st);
            }
            cudaEvent_t ej;
            cudaEventCreateWithFlags(&ej, cudaEventDisableTiming);
            cudaEventRecord(ej, s1);
            cudaStreamWaitEvent(s0, ej, 0);
            cudaEventDestroy(ej);
        }, bytes / 1e6);
    }
    timeit("memcpy D2H 1 MB", [&] { cudaMemcpyAsync(ho, d, obytes, cudaMemcpyDeviceToHost, s0); }, obytes / 1e6);
    for (int g : {1, 2, 4, 8}) {
        char name[64];
        std::snprintf(name, sizeof name, "zero-copy read u32, %d CTAs/SM", g);
        timeit(name, [&] { zc_read<uint32_t><<<sms * g, 256, 0, s0>>>((const uint32_t *)hd, bytes / 4, out); }, bytes / 1e6);
    }
    timeit("zero-copy read u64, 8 CTAs/SM", [&] { zc_read<uint2><<<sms * 8, 256, 0, s0>>>((const uint2 *)hd, bytes / 8, out); }, bytes / 1e6);
    timeit("zero-copy read 16B, 8 CTAs/SM", [&] { zc_read<uint4><<<sms * 8, 256, 0, s0>>>((const uint4 *)hd, bytes / 16, out); }, bytes / 1e6);
    timeit("zero-copy write 1 MB", [&] { zc_write<<<sms * 4, 256, 0, s0>>>((uint8_t *)hod, obytes); }, obytes / 1e6);
    timeit("zero-copy read 8 MB + write 1 MB (2 streams)", [&] {
        cudaEvent_t es;
        cudaEventCreateWithFlags(&es, cudaEventDisableTiming);
        cudaEventRecord(es, s0);
        cudaStreamWaitEvent(s1, es, 0);
        cudaEventDestroy(es);
        zc_write<<<sms * 2, 256, 0, s1>>>((uint8_t *)hod, obytes);
        zc_read<uint32_t><<<sms * 6, 256, 0, s0>>>((const uint32_t *)hd, bytes / 4, out);
        cudaEvent_t ej;
        cudaEventCreateWithFlags(&ej, cudaEventDisableTiming);
        cudaEventRecord(ej, s1);
        cudaStreamWaitEvent(s0, ej, 0);
        cudaEventDestroy(ej);
    }, (bytes + obytes) / 1e6);
    // hybrid: a share of the 8 MB read zero-copy by a kernel while the copy
    // engine moves the rest (both on the same link)
    for (int pct : {30, 40, 50, 60}) {
        const size_t zc = (bytes * pct / 100) & ~(size_t)255;
        char name[64];
        std::snprintf(name, sizeof name, "hybrid: %d%% zero-copy + rest by DMA", pct);
        timeit(name, [&] {
            cudaEvent_t es;
            cudaEventCreateWithFlags(&es, cudaEventDisableTiming);
            cudaEventRecord(es, s0);
            cudaStreamWaitEvent(s1, es, 0);
            cudaEventDestroy(es);
            cudaMemcpyAsync((char *)d + zc, (char *)h + zc, bytes - zc, cudaMemcpyHostToDevice, s1);
            zc_read<uint4><<<sms * 4, 256, 0, s0>>>((const uint4 *)hd, zc / 16, out);
            cudaEvent_t ej;
            cudaEventCreateWithFlags(&ej, cudaEventDisableTiming);
            cudaEventRecord(ej, s1);
            cudaStreamWaitEvent(s0, ej, 0);
            cudaEventDestroy(ej);
        }, bytes / 1e6);
    }
    return 0;
}
