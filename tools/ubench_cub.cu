// Host-side cost of CUB dispatch for insert-batch-sized inputs (100k keys):
// the temp-size query and the enqueue of SortKeys / Unique / ExclusiveSum,
// without waiting for the GPU (the insert path is host-bound).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_cub tools/ubench_cub.cu
#include <cub/cub.cuh>
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>

template <typename F>
static double med_us(F f, int n = 200) {
    std::vector<double> t;
    for (int i = 0; i < n; ++i) {
        auto a = std::chrono::steady_clock::now();
        f();
        auto b = std::chrono::steady_clock::now();
        t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
        cudaDeviceSynchronize();
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

__global__ void tiny(int *p) { if (p && threadIdx.x == 1234) *p = 0; }

int main() {
    const int N = 100000;
    uint64_t *a, *b, *c;
    uint32_t *x, *y;
    cudaMalloc(&a, N * 8); cudaMalloc(&b, N * 8); cudaMalloc(&c, N * 8);
    cudaMalloc(&x, (1 << 20) * 4 + 64); cudaMalloc(&y, (1 << 20) * 4 + 64);
    cudaMemset(a, 0, N * 8);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    void *tmp = nullptr;
    cudaMalloc(&tmp, 64 << 20);
    size_t tb = 0;
    cub::DoubleBuffer<uint64_t> db(a, b);
    std::printf("kernel launch (enqueue only)          %6.2f us\n", med_us([&] { tiny<<<1, 32, 0, s>>>(nullptr); }));
    std::printf("cudaMemsetAsync 4 MB (enqueue)         %6.2f us\n", med_us([&] { cudaMemsetAsync(x, 0, 4 << 20, s); }));
    std::printf("SortKeys size query                    %6.2f us\n", med_us([&] { cub::DeviceRadixSort::SortKeys(nullptr, tb, db, N, 0, 40, s); }));
    std::printf("SortKeys enqueue (40-bit keys)         %6.2f us\n", med_us([&] { size_t t = 64 << 20; cub::DeviceRadixSort::SortKeys(tmp, t, db, N, 0, 40, s); }));
    std::printf("Unique size query                      %6.2f us\n", med_us([&] { cub::DeviceSelect::Unique(nullptr, tb, a, c, (uint64_t *)x, N, s); }));
    std::printf("Unique enqueue                         %6.2f us\n", med_us([&] { size_t t = 64 << 20; cub::DeviceSelect::Unique(tmp, t, a, c, (uint64_t *)x, N, s); }));
    std::printf("ExclusiveSum size query (2^20+1)       %6.2f us\n", med_us([&] { cub::DeviceScan::ExclusiveSum(nullptr, tb, x, y, (1 << 20) + 1, s); }));
    std::printf("ExclusiveSum enqueue (2^20+1)          %6.2f us\n", med_us([&] { size_t t = 64 << 20; cub::DeviceScan::ExclusiveSum(tmp, t, x, y, (1 << 20) + 1, s); }));
    return 0;
}
