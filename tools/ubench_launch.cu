// Fixed cost of one kernel launch as the bench's events see it: an empty
// 1184 x 256 kernel between two events, queued behind a ~50 us busy kernel
// so the host launch latency is hidden (as in bench.py, where the L2 flush
// runs ahead of the query kernel).  Built twice:
//   plain: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_launch tools/ubench_launch.cu
//   rdc:   ... -DWITH_TAIL -rdc=true -o tools/ubench_launch_rdc tools/ubench_launch.cu -lcudadevrt
// The rdc build's kernel holds a (never taken) cudaStreamTailLaunch, like
// label_lean_kernel; the difference is the device-runtime launch overhead.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void busy_kernel(unsigned long long ns) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > ns) break;
    }
}

__global__ void child_kernel() {}

struct Big { unsigned long long w[20]; };

__global__ void empty_kernel(int *flag, Big b) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && *flag == 12345 && b.w[3] == 7) {
#ifdef WITH_TAIL
        child_kernel<<<1, 32, 0, cudaStreamTailLaunch>>>();
#else
        *flag = 0;
#endif
    }
}

__global__ void small_kernel(int *flag) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && *flag == 12345) *flag = 0;
}

int main() {
    int *flag;
    cudaMalloc(&flag, 4);
    cudaMemset(flag, 0, 4);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    Big b{};
    for (int variant = 0; variant < 4; ++variant) {
        std::vector<float> ts;
        for (int i = 0; i < 220; ++i) {
            busy_kernel<<<1, 32, 0, s>>>(50000);
            cudaEventRecord(e0, s);
            if (variant == 0) small_kernel<<<1184, 256, 0, s>>>(flag);
            else if (variant == 1) empty_kernel<<<1184, 256, 0, s>>>(flag, b);
            else if (variant == 2) { small_kernel<<<1184, 256, 0, s>>>(flag); small_kernel<<<1184, 256, 0, s>>>(flag); }
            else { cudaEventRecord(e1, s); }
            if (variant != 3) cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (i >= 20) ts.push_back(ms * 1e3f);
        }
        std::sort(ts.begin(), ts.end());
        double mean = 0;
        for (float t : ts) mean += t;
        mean /= ts.size();
        const char *names[] = {"small kernel (8B param)", "empty kernel (160B param"
#ifdef WITH_TAIL
                               ", tail-launch capable, rdc)",
#else
                               ", plain)",
#endif
                               "two small kernels", "no kernel (event pair)"};
        std::printf("%-50s median %6.2f us  mean %6.2f us\n", names[variant], ts[ts.size() / 2], mean);
    }
    // the same empty kernel as a one-node CUDA graph
    {
        cudaGraph_t gr;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        small_kernel<<<1184, 256, 0, s>>>(flag);
        cudaStreamEndCapture(s, &gr);
        cudaGraphInstantiate(&ge, gr, 0);
        std::vector<float> ts;
        for (int i = 0; i < 220; ++i) {
            busy_kernel<<<1, 32, 0, s>>>(50000);
            cudaEventRecord(e0, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (i >= 20) ts.push_back(ms * 1e3f);
        }
        std::sort(ts.begin(), ts.end());
        std::printf("small kernel as a CUDA graph                      median %6.2f us\n", ts[ts.size() / 2]);
    }
    // programmatic dependent launch after the busy kernel (the event pair still around it)
    {
        std::vector<float> ts;
        for (int i = 0; i < 220; ++i) {
            busy_kernel<<<1, 32, 0, s>>>(50000);
            cudaEventRecord(e0, s);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(1184);
            cfg.blockDim = dim3(256);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, small_kernel, flag);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (i >= 20) ts.push_back(ms * 1e3f);
        }
        std::sort(ts.begin(), ts.end());
        std::printf("small kernel with PDL attribute                   median %6.2f us\n", ts[ts.size() / 2]);
    }
    // CTA count vs fixed cost: same thread count, different CTA sizes
    const int cfgs[][2] = {{1184, 256}, {592, 512}, {296, 1024}, {148, 1024}, {2368, 128}, {148, 256}};
    for (auto &c : cfgs) {
        std::vector<float> ts;
        for (int i = 0; i < 220; ++i) {
            busy_kernel<<<1, 32, 0, s>>>(50000);
            cudaEventRecord(e0, s);
            small_kernel<<<c[0], c[1], 0, s>>>(flag);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (i >= 20) ts.push_back(ms * 1e3f);
        }
        std::sort(ts.begin(), ts.end());
        std::printf("small kernel %5d x %4d                          median %6.2f us\n", c[0], c[1], ts[ts.size() / 2]);
    }
    return 0;
}
