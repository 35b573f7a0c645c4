// Library comparison point on the same B200: CUB's DeviceRadixSort (the
// onesweep implementation shipped with CUDA 12.9) on the bench workloads.
// Not part of the product; it answers "how does the hand-written onesweep
// compare with the vendor library on this GPU".
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        tools/cub_compare.cu -o build/cub_compare && build/cub_compare
//
// Prints one JSON line per case: ms per sort (CUDA events, median of 10
// after 3 warm-ups, inputs resident, > L2), keys/s and the bytes a 4 x 8-bit
// LSD sort moves (the same algorithmic figure bench.py divides by).
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 1;                                                            \
        }                                                                        \
    } while (0)

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// kind 0: uniform 32-bit; 1: ascending; 2: uniform 64-bit key + index payload
__global__ void fill(uint32_t* k32, unsigned long long* k64, uint32_t* v, size_t n, int kind) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const uint64_t z = splitmix(i * 0x9E3779B97F4A7C15ull + 1);
        if (kind == 0) k32[i] = (uint32_t)(z >> 32);
        if (kind == 1) k32[i] = (uint32_t)i;
        if (kind == 2) {
            k64[i] = z;
            v[i] = (uint32_t)i;
        }
    }
}

template <typename S, typename F>
static float median_ms(S&& setup, F&& f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) {
        setup();
        f();
    }
    std::vector<float> t;
    for (int i = 0; i < 10; ++i) {
        setup();  // fresh unsorted input every rep, outside the timed region
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    const size_t n = 1ull << 28;
    uint32_t *k32a, *k32b, *va, *vb;
    unsigned long long *k64a, *k64b;
    CK(cudaMalloc(&k32a, n * 4));
    CK(cudaMalloc(&k32b, n * 4));
    CK(cudaMalloc(&va, n * 4));
    CK(cudaMalloc(&vb, n * 4));
    CK(cudaMalloc(&k64a, n * 8));
    CK(cudaMalloc(&k64b, n * 8));
    void* tmp = nullptr;
    size_t tb = 0, t2 = 0;
    {
        cub::DoubleBuffer<uint32_t> d(k32a, k32b);
        CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, d, (int)n));
        cub::DoubleBuffer<unsigned long long> dk(k64a, k64b);
        cub::DoubleBuffer<uint32_t> dv(va, vb);
        CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, dk, dv, (int)n));
        tb = std::max(tb, t2);
    }
    CK(cudaMalloc(&tmp, tb));

    struct Case {
        const char* name;
        int kind;
        size_t n;
    } cases[] = {{"cfg2 u32 uniform 2^28", 0, n},
                 {"u32 ascending 2^27", 1, n / 2},
                 {"cfg5 u64 key + u32 payload 2^28", 2, n}};
    for (const Case& c : cases) {
        float ms;
        double bytes;
        if (c.kind < 2) {
            ms = median_ms([&] { fill<<<1184, 256>>>(k32a, nullptr, nullptr, c.n, c.kind); }, [&] {
                cub::DoubleBuffer<uint32_t> d(k32a, k32b);
                size_t t = tb;
                cub::DeviceRadixSort::SortKeys(tmp, t, d, (int)c.n);
            });
            bytes = 4.0 * 2 * 4 * c.n;
        } else {
            ms = median_ms([&] { fill<<<1184, 256>>>(nullptr, k64a, va, c.n, 2); }, [&] {
                cub::DoubleBuffer<unsigned long long> dk(k64a, k64b);
                cub::DoubleBuffer<uint32_t> dv(va, vb);
                size_t t = tb;
                cub::DeviceRadixSort::SortPairs(tmp, t, dk, dv, (int)c.n);
            });
            bytes = 8.0 * 2 * 12 * c.n;
        }
        CK(cudaGetLastError());
        printf("{\"impl\": \"cub\", \"cub_version\": %d, \"case\": \"%s\", \"n\": %zu, \"ms\": %.4f, "
               "\"keys_per_s\": %.4g, \"lsd_pass_bytes_GBps\": %.1f}\n",
               CUB_VERSION, c.name, c.n, ms, c.n / (ms * 1e-3), bytes / (ms * 1e-3) / 1e9);
    }
    return 0;
}
