// Cost of a cooperative-groups grid barrier on this part, by grid size.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_gridsync tools/ubench_gridsync.cu
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void syncs(int iters, unsigned *sink) {
    cg::grid_group grid = cg::this_grid();
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += threadIdx.x ^ i;
        grid.sync();
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *sink;
    cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int threads : {256, 512}) {
        for (int bps : {1, 2, 4, 8}) {
            if (threads * bps > 2048) continue;
            const int grid = sms * bps;
            float t[2];
            for (int k = 0; k < 2; ++k) {
                int iters = k ? 1001 : 1;
                void *args[] = {(void *)&iters, (void *)&sink};
                cudaLaunchCooperativeKernel((const void *)syncs, dim3(grid), dim3(threads), args, 0, 0);
                cudaEventRecord(e0);
                cudaLaunchCooperativeKernel((const void *)syncs, dim3(grid), dim3(threads), args, 0, 0);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&t[k], e0, e1);
            }
            std::printf("threads %4d  CTAs %5d  launch %6.1f us  per grid.sync %5.2f us  (%s)\n", threads, grid,
                        t[0] * 1e3, (t[1] - t[0]) * 1e3 / 1000.0, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
