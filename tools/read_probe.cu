// Read-only HBM ceiling on this B200: one streaming read of 1 GiB with 16-byte
// loads (8 in flight per thread, one wave of 1024-thread CTAs, like the
// all-digit prologue) and a copy of 1 GiB, timed with CUDA events (median of
// 10). The prologue's roofline is the read figure, the passes' the copy one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/read_probe.cu -o build/read_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void __launch_bounds__(1024, 1) read_kernel(const uint4* __restrict__ p, size_t nvec,
                                                      unsigned* __restrict__ sink) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned acc = 0;
    size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; v + 7 * stride < nvec; v += 8 * stride) {
        uint4 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = __ldcs(p + v + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= q[u].x ^ q[u].y ^ q[u].z ^ q[u].w;
    }
    for (; v < nvec; v += stride) {
        const uint4 q = __ldcs(p + v);
        acc ^= q.x ^ q.y ^ q.z ^ q.w;
    }
    if (acc == 0x9e3779b9u) *sink = acc;
}

int main() {
    const size_t bytes = 1ull << 30;
    uint4 *a, *b;
    unsigned* sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto med = [&](auto f) {
        std::vector<float> t;
        for (int i = 0; i < 13; ++i) {
            cudaEventRecord(e0);
            f();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (i >= 3) t.push_back(ms);
        }
        std::sort(t.begin(), t.end());
        return t[t.size() / 2];
    };
    const float r = med([&] { read_kernel<<<sms, 1024>>>(a, bytes / 16, sink); });
    const float c = med([&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); });
    printf("{\"read_1GiB_ms\": %.4f, \"read_GBps\": %.1f, \"copy_1GiB_ms\": %.4f, \"copy_GBps_rw\": %.1f}\n", r,
           bytes / (r * 1e-3) / 1e9, c, 2 * bytes / (c * 1e-3) / 1e9);
    return 0;
}
