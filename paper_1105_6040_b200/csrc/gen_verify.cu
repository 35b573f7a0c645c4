// gen_verify.cu -- device input generator and output verifier.
//
// gen_keys_kernel restates bench::gen_data (P/src/bench.cpp:57-71) in closed
// form: element i of the splitmix64 stream is mix(seed + (i+1)*gamma), so any
// window of the stream is generated in parallel, bit-identical to the host.
// check_sorted_kernel is the device form of bench::verify_output's gate
// (P/src/bench.cpp:95-104, kernels::is_sorted P/src/sort_core.cpp:146-151):
// it counts adjacent inversions and returns the golden fixtures' fingerprint
// and an order-independent multiset hash, so a 2^31-key output is checked
// without a host round trip.
#include <cub/block/block_reduce.cuh>

#include "b2s_internal.cuh"

namespace b2s {
namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

template <typename T>
__global__ void gen_keys_kernel(uint64_t first, uint64_t n, uint64_t seed, int shift,
                                T* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t z = mix64(seed + (first + i + 1) * kGamma);
        out[i] = (T)(z >> shift);
    }
}

// cfg4a's Zipf stream: u = z_i >> 11 (53 bits) of
// gen_data's element i, key = number of thresholds <= u (the rank drawn by the
// integer inverse-CDF table, see oracle.zipf_thresholds). Integer only, so the
// device and the host draw identical keys from the same table.
template <typename T>
__global__ void gen_zipf_kernel(uint64_t first, uint64_t n, uint64_t seed,
                                const uint64_t* __restrict__ t, uint32_t nv, T* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t u = mix64(seed + (first + i + 1) * kGamma) >> 11;
        uint32_t lo = 0, hi = nv;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(t + mid) <= u) lo = mid + 1;
            else hi = mid;
        }
        out[i] = (T)lo;
    }
}

template <typename T>
__device__ __forceinline__ uint64_t widen(T x) {
    return (uint64_t)(int64_t)x;  // sign-extends signed types, zero-extends unsigned
}
template <>
__device__ __forceinline__ uint64_t widen<uint32_t>(uint32_t x) {
    return (uint64_t)x;
}

template <typename T>
__global__ void __launch_bounds__(256) check_sorted_kernel(const T* __restrict__ k, uint64_t n,
                                                           unsigned long long* __restrict__ acc) {
    using BR = cub::BlockReduce<unsigned long long, 256>;
    __shared__ typename BR::TempStorage tmp;
    unsigned long long inv = 0, fp = 0, ms = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const T x = k[i];
        if (i > 0 && k[i - 1] > x) ++inv;
        const uint64_t w = widen(x);
        fp += mix64(w ^ mix64(i + 1));
        ms += mix64(w);
    }
    unsigned long long r = BR(tmp).Sum(inv);
    if (threadIdx.x == 0) atomicAdd(&acc[0], r);
    __syncthreads();
    r = BR(tmp).Sum(fp);
    if (threadIdx.x == 0) atomicAdd(&acc[1], r);
    __syncthreads();
    r = BR(tmp).Sum(ms);
    if (threadIdx.x == 0) atomicAdd(&acc[2], r);
}

}  // namespace

b2s_status gen_keys(b2s_ctx* ctx, b2s_dtype dtype, uint64_t first, uint64_t n, uint64_t seed,
                    int shift, void* out) {
    if (n == 0) return B2S_OK;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->num_sms * 16);
    switch (dtype) {
        case B2S_I32:
            gen_keys_kernel<int32_t><<<grid, 256, 0, ctx->stream>>>(first, n, seed, shift,
                                                                    static_cast<int32_t*>(out));
            break;
        case B2S_U32:
            gen_keys_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(first, n, seed, shift,
                                                                     static_cast<uint32_t*>(out));
            break;
        case B2S_I64:
            gen_keys_kernel<int64_t><<<grid, 256, 0, ctx->stream>>>(first, n, seed, shift,
                                                                    static_cast<int64_t*>(out));
            break;
        case B2S_U64:
            gen_keys_kernel<unsigned long long><<<grid, 256, 0, ctx->stream>>>(
                first, n, seed, shift, static_cast<unsigned long long*>(out));
            break;
    }
    B2S_LAUNCHED();
    return B2S_OK;
}

b2s_status gen_zipf(b2s_ctx* ctx, b2s_dtype dtype, uint64_t first, uint64_t n, uint64_t seed,
                    const uint64_t* thresholds, uint32_t nvalues, void* out) {
    if (n == 0) return B2S_OK;
    B2S_TRY(ctx->zipf_table.ensure((size_t)nvalues * 8));
    uint64_t* t = static_cast<uint64_t*>(ctx->zipf_table.ptr);
    B2S_CUDA(cudaMemcpyAsync(t, thresholds, (size_t)nvalues * 8, cudaMemcpyHostToDevice, ctx->stream));
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->num_sms * 16);
    switch (dtype) {
        case B2S_I32:
            gen_zipf_kernel<int32_t><<<grid, 256, 0, ctx->stream>>>(first, n, seed, t, nvalues,
                                                                    static_cast<int32_t*>(out));
            break;
        case B2S_U32:
            gen_zipf_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(first, n, seed, t, nvalues,
                                                                     static_cast<uint32_t*>(out));
            break;
        case B2S_I64:
            gen_zipf_kernel<int64_t><<<grid, 256, 0, ctx->stream>>>(first, n, seed, t, nvalues,
                                                                    static_cast<int64_t*>(out));
            break;
        case B2S_U64:
            gen_zipf_kernel<unsigned long long><<<grid, 256, 0, ctx->stream>>>(
                first, n, seed, t, nvalues, static_cast<unsigned long long*>(out));
            break;
    }
    B2S_LAUNCHED();
    // the table is pageable host memory: the copy is staged before the call
    // returns, so the caller may free it
    return B2S_OK;
}

b2s_status check_sorted(b2s_ctx* ctx, b2s_dtype dtype, const void* keys, uint64_t n,
                        uint64_t* inv, uint64_t* fp, uint64_t* ms) {
    B2S_TRY(ctx->misc.ensure(64));
    B2S_TRY(ctx->host_misc.ensure(64));
    unsigned long long* acc = static_cast<unsigned long long*>(ctx->misc.ptr);
    B2S_CUDA(cudaMemsetAsync(acc, 0, 3 * sizeof(unsigned long long), ctx->stream));
    const unsigned grid =
        (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->num_sms * 8));
    switch (dtype) {
        case B2S_I32:
            check_sorted_kernel<int32_t><<<grid, 256, 0, ctx->stream>>>(
                static_cast<const int32_t*>(keys), n, acc);
            break;
        case B2S_U32:
            check_sorted_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(
                static_cast<const uint32_t*>(keys), n, acc);
            break;
        case B2S_I64:
            check_sorted_kernel<int64_t><<<grid, 256, 0, ctx->stream>>>(
                static_cast<const int64_t*>(keys), n, acc);
            break;
        case B2S_U64:
            check_sorted_kernel<unsigned long long><<<grid, 256, 0, ctx->stream>>>(
                static_cast<const unsigned long long*>(keys), n, acc);
            break;
    }
    B2S_LAUNCHED();
    B2S_CUDA(cudaMemcpyAsync(ctx->host_misc.ptr, acc, 3 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, ctx->stream));
    B2S_CUDA(cudaStreamSynchronize(ctx->stream));
    const unsigned long long* h = static_cast<const unsigned long long*>(ctx->host_misc.ptr);
    if (inv) *inv = h[0];
    if (fp) *fp = h[1];
    if (ms) *ms = h[2];
    return B2S_OK;
}

}  // namespace b2s
