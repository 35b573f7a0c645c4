// sample_sort.cu -- device steps of the multi-GPU sample sort.
//
// Replaces the reference's data distribution (Comm::scatter/gather and the p
// odd-even block exchanges, P/src/runtime.cpp:509-568,
// P/src/parallel_sort.cpp:188-248) across GPUs. Each GPU (one process per GPU)
// holds a contiguous shard (plan_partition, P/src/parallel_sort.cpp:26-38),
// sorts it, and then:
//   sample_regular_kernel   s regular samples of the sorted shard as compound
//                           (key, rank, sorted position) records
//   [host: all-gather of the samples over NCCL]
//   select_splitters_kernel 1 CTA: bitonic sort of all samples in shared
//                           memory, splitter i = sample at rank i*m/G
//   bucket_bounds_kernel    per splitter, the number of local keys ordered
//                           before it in (key, rank, position) order: a
//                           binary search, or the sample's own position
//   [host: all-to-all of the buckets over NCCL, k-way merge of received runs]
// Compound keys make every record distinct, so equal keys (cfg4 all-equal,
// Zipf) still split evenly and the result is stable by global index.
#include "b2s_internal.cuh"

namespace b2s {
namespace {

constexpr uint64_t kEmpty = ~0ull;

template <typename U>
__device__ __forceinline__ uint64_t ord_bits(U k, U sign) {
    return (uint64_t)(k ^ sign);
}

template <typename U>
__global__ void sample_regular_kernel(const U* __restrict__ keys, uint64_t n, int rank, int s,
                                      U sign, b2s_sample* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= s) return;
    if (n == 0) {
        out[j] = {kEmpty, kEmpty};
        return;
    }
    // centred regular positions (2j+1) n / 2s
    const uint64_t pos = (uint64_t)(((unsigned __int128)(2 * (uint64_t)j + 1) * n) / (2 * (uint64_t)s));
    out[j] = {ord_bits(keys[pos], sign), ((uint64_t)rank << 40) | pos};
}

__device__ __forceinline__ bool sample_less(const b2s_sample& a, const b2s_sample& b) {
    return a.key < b.key || (a.key == b.key && a.tag < b.tag);
}

constexpr int kSelectMax = 8192;  // samples sorted in one CTA

__global__ void __launch_bounds__(1024) select_splitters_kernel(const b2s_sample* __restrict__ in,
                                                                int count, int nparts,
                                                                b2s_sample* __restrict__ out) {
    extern __shared__ b2s_sample s[];
    __shared__ int s_valid;
    int m = 1;
    while (m < count) m <<= 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) s[i] = i < count ? in[i] : b2s_sample{kEmpty, kEmpty};
    if (threadIdx.x == 0) s_valid = 0;
    __syncthreads();
    // bitonic sort, ascending
    for (int k = 2; k <= m; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const bool up = (i & k) == 0;
                    const b2s_sample a = s[i], b = s[p];
                    if (sample_less(b, a) == up) {
                        s[i] = b;
                        s[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    int local = 0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) local += s[i].tag != kEmpty;
    atomicAdd(&s_valid, local);
    __syncthreads();
    const int v = s_valid;
    for (int i = threadIdx.x; i + 1 < nparts; i += blockDim.x) {
        const int r = (int)(((long long)(i + 1) * v) / nparts);
        out[i] = v > 0 ? s[r < v ? r : v - 1] : b2s_sample{kEmpty, kEmpty};
    }
}

template <typename U>
__device__ uint64_t lower_upper(const U* keys, uint64_t n, uint64_t key, U sign, bool upper) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const uint64_t k = ord_bits(keys[mid], sign);
        if (k < key || (upper && k == key)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename U>
__global__ void bucket_bounds_kernel(const U* __restrict__ keys, uint64_t n, int rank, U sign,
                                     const b2s_sample* __restrict__ spl, int nparts,
                                     uint64_t* __restrict__ bounds) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > nparts) return;
    if (i == 0) {
        bounds[0] = 0;
        return;
    }
    if (i == nparts) {
        bounds[nparts] = n;
        return;
    }
    const b2s_sample s = spl[i - 1];
    uint64_t c;
    if (s.tag == kEmpty) {
        c = n;
    } else {
        const int srank = (int)(s.tag >> 40);
        if (rank < srank) c = lower_upper(keys, n, s.key, sign, true);
        else if (rank > srank) c = lower_upper(keys, n, s.key, sign, false);
        else c = s.tag & ((1ull << 40) - 1);
    }
    bounds[i] = c;
}

}  // namespace

b2s_status sample_regular(b2s_ctx* ctx, b2s_dtype dtype, const void* keys, uint64_t n, int rank,
                          int s, b2s_sample* out) {
    const unsigned grid = (unsigned)((s + 255) / 256);
    switch (dtype) {
        case B2S_I32:
        case B2S_U32:
            sample_regular_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(
                static_cast<const uint32_t*>(keys), n, rank, s,
                dtype == B2S_I32 ? 0x80000000u : 0u, out);
            break;
        default:
            sample_regular_kernel<unsigned long long><<<grid, 256, 0, ctx->stream>>>(
                static_cast<const unsigned long long*>(keys), n, rank, s,
                dtype == B2S_I64 ? (1ull << 63) : 0ull, out);
    }
    B2S_LAUNCHED();
    return B2S_OK;
}

b2s_status select_splitters(b2s_ctx* ctx, const b2s_sample* samples, int count, int nparts,
                            b2s_sample* splitters) {
    if (count > kSelectMax)
        return set_error(B2S_EINVAL, "select_splitters: %d samples exceed %d", count, kSelectMax);
    if (nparts < 2) return B2S_OK;
    int m = 1;
    while (m < count) m <<= 1;
    const size_t smem = (size_t)m * sizeof(b2s_sample);
    static DeviceOnce once;
    B2S_TRY(once_per_device(once, ctx->device, [&]() -> b2s_status {
        B2S_CUDA(cudaFuncSetAttribute(select_splitters_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(kSelectMax * sizeof(b2s_sample))));
        return B2S_OK;
    }));
    select_splitters_kernel<<<1, 1024, smem, ctx->stream>>>(samples, count, nparts, splitters);
    B2S_LAUNCHED();
    return B2S_OK;
}

b2s_status bucket_bounds(b2s_ctx* ctx, b2s_dtype dtype, const void* keys, uint64_t n, int rank,
                         const b2s_sample* splitters, int nparts, uint64_t* bounds) {
    const unsigned grid = (unsigned)((nparts + 1 + 255) / 256);
    switch (dtype) {
        case B2S_I32:
        case B2S_U32:
            bucket_bounds_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(
                static_cast<const uint32_t*>(keys), n, rank,
                dtype == B2S_I32 ? 0x80000000u : 0u, splitters, nparts, bounds);
            break;
        default:
            bucket_bounds_kernel<unsigned long long><<<grid, 256, 0, ctx->stream>>>(
                static_cast<const unsigned long long*>(keys), n, rank,
                dtype == B2S_I64 ? (1ull << 63) : 0ull, splitters, nparts, bounds);
    }
    B2S_LAUNCHED();
    return B2S_OK;
}

}  // namespace b2s
