// Cost of the fixpoint compaction's slot reservation: every warp does R
// rounds of {one 64-bit atomicAdd with return on ONE global counter, then a
// shuffle of the result}, rounds serial (as in compact_bitmap), at the
// fixpoint's grid (148 x 4 CTAs x 256 threads).  Compares 1 counter vs the
// same work spread over 8 / 64 counters, and the no-return reduction.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_atomic tools/ubench_atomic.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <bool RET>
__global__ void rounds(unsigned long long *cnt, int ncnt, int R, unsigned long long *sink) {
    const int lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned long long acc = 0;
    for (int r = 0; r < R; ++r) {
        unsigned long long base = 0;
        if (lane == 31) {
            if (RET) base = atomicAdd(cnt + (warp % ncnt) * 16, (87ull << 32) | 120ull);
            else atomicAdd(cnt + (warp % ncnt) * 16, (87ull << 32) | 120ull);
        }
        base = __shfl_sync(0xffffffffu, base, 31);
        acc += base;
    }
    if (acc == 12345) *sink = acc;
}

int main() {
    unsigned long long *cnt, *sink;
    cudaMalloc(&cnt, 64 * 16 * 8);
    cudaMalloc(&sink, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int R : {14, 28}) {
        for (int nc : {1, 8, 64}) {
            for (int ret = 1; ret >= 0; --ret) {
                float best = 1e9f;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaMemset(cnt, 0, 64 * 16 * 8);
                    cudaEventRecord(a);
                    if (ret) rounds<true><<<sms * 4, 256>>>(cnt, nc, R, sink);
                    else rounds<false><<<sms * 4, 256>>>(cnt, nc, R, sink);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (rep && ms < best) best = ms;
                }
                const double n = (double)sms * 4 * 8 * R;
                printf("R=%2d counters=%2d %s: %8.1f us  (%.2f ns per atomic)\n", R, nc, ret ? "atomicAdd" : "red      ",
                       best * 1e3, best * 1e6 / n);
            }
        }
    }
    return 0;
}
