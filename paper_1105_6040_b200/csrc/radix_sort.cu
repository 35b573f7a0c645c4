// radix_sort.cu -- LSD onesweep radix sort for sm_100a.
//
// Replaces the reference's per-rank comparison sorts (kernels::merge_sort /
// quick_sort / bubble_sort, P/src/sort_core.cpp:23-144, reached through
// KernelFn, P/src/parallel_sort.cpp:136-164). The output is the same ascending
// array std::sort gives (P/src/bench.cpp:95-104); with a payload the sort is
// stable (equal keys keep input order, merge_sort's tie rule :77).
//
// Structure (one call, all on one stream, no host round trip):
//   radix_hist_kernel   one read of the keys: 256-bin histograms of EVERY
//                       8-bit digit position at once, and zeroes look-back
//                       region 0.
//   radix_plan_kernel   1 CTA: exclusive scan per digit position -> global
//                       digit offsets; marks constant digits (one bin holds
//                       all n keys) as skipped; assigns ping-pong buffers so
//                       the last executed pass lands in the output.
//   onesweep_kernel x S one launch per digit slot: persistent CTAs take tiles
//                       from an atomic counter, rank keys in-warp with
//                       __match_any_sync, publish per-digit tile counts, resolve
//                       the tile's global offsets by decoupled look-back, stage
//                       the tile digit-sorted in shared memory, and write runs
//                       of equal digits with coalesced stores.
//   radix_copy_kernel   only does work when an in-place sort executed an odd
//                       number of passes (or zero passes out of place).
//
// HBM traffic per executed pass: read + write of every key (and payload):
// 2 * (key_bytes + val_bytes) * n. The histogram reads key_bytes * n once.
#include <cub/warp/warp_scan.cuh>

#include <stdlib.h>

#include "b2s_internal.cuh"

namespace b2s {
namespace {

constexpr int kRadix = 256;

template <typename LB>
struct LookbackWord;
template <>
struct LookbackWord<uint32_t> {
    static constexpr uint32_t kAgg = 1u << 30, kInc = 2u << 30, kMask = (1u << 30) - 1;
    static __device__ __forceinline__ uint32_t flag(uint32_t w) { return w >> 30; }
};
template <>
struct LookbackWord<unsigned long long> {
    static constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62,
                                        kMask = (1ull << 62) - 1;
    static __device__ __forceinline__ unsigned long long flag(unsigned long long w) {
        return w >> 62;
    }
};

__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <typename U>
__device__ __forceinline__ uint32_t digit_of(U k, int shift, uint32_t dxor) {
    return ((uint32_t)(k >> shift) & 0xFFu) ^ dxor;
}

// ---------------------------------------------------------------------------
// upfront histogram of all digit positions

template <typename U>
__global__ void __launch_bounds__(512) radix_hist_kernel(const U* __restrict__ keys, uint64_t n,
                                                         uint32_t top_xor,
                                                         unsigned long long* __restrict__ g_hist,
                                                         uint4* __restrict__ lb_zero,
                                                         uint64_t lb_zero_vecs) {
    constexpr int NP = sizeof(U);
    constexpr int VEC = 16 / sizeof(U);
    __shared__ uint32_t s_h[NP][kRadix];
    for (int i = threadIdx.x; i < NP * kRadix; i += blockDim.x) (&s_h[0][0])[i] = 0;
    __syncthreads();

    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;

    for (uint64_t i = tid; i < lb_zero_vecs; i += stride) lb_zero[i] = make_uint4(0, 0, 0, 0);

    // run-length aggregation per digit position: sorted / constant inputs
    // collapse to a few shared-memory atomics instead of one per key
    uint32_t cur[NP], cnt[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        cur[p] = 0;
        cnt[p] = 0;
    }
    auto count_key = [&](U k) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            uint32_t d = (uint32_t)(k >> (8 * p)) & 0xFFu;
            if (p == NP - 1) d ^= top_xor;
            if (d == cur[p]) {
                ++cnt[p];
            } else {
                if (cnt[p]) atomicAdd(&s_h[p][cur[p]], cnt[p]);
                cur[p] = d;
                cnt[p] = 1;
            }
        }
    };

    const uint64_t nvec = n / VEC;
    const uint4* kv = reinterpret_cast<const uint4*>(keys);
    const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
    if (aligned) {
        for (uint64_t v = tid; v < nvec; v += stride) {
            uint4 q = __ldcs(kv + v);
            const U* e = reinterpret_cast<const U*>(&q);
#pragma unroll
            for (int j = 0; j < VEC; ++j) count_key(e[j]);
        }
        for (uint64_t i = nvec * VEC + tid; i < n; i += stride) count_key(keys[i]);
    } else {
        for (uint64_t i = tid; i < n; i += stride) count_key(keys[i]);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p)
        if (cnt[p]) atomicAdd(&s_h[p][cur[p]], cnt[p]);
    __syncthreads();
    for (int i = threadIdx.x; i < NP * kRadix; i += blockDim.x) {
        const uint32_t c = (&s_h[0][0])[i];
        if (c) atomicAdd(&g_hist[i], (unsigned long long)c);
    }
}

// ---------------------------------------------------------------------------
// pass plan: global digit offsets, skipped digits, buffer chain

__global__ void __launch_bounds__(256) radix_plan_kernel(
    RadixPlan* __restrict__ plan, unsigned long long* __restrict__ g_hist, int np, uint64_t n,
    uint32_t top_xor, const void* kin, void* kout, void* ktmp, const uint32_t* vin,
    uint32_t* vout, uint32_t* vtmp) {
    using WarpScan = cub::WarpScan<unsigned long long>;
    __shared__ typename WarpScan::TempStorage ws[8];
    __shared__ unsigned long long s_warp[8];
    __shared__ int s_trivial[kMaxSlots];
    const int d = threadIdx.x, warp = d >> 5, lane = d & 31;

    for (int p = 0; p < np; ++p) {
        const unsigned long long c = g_hist[p * kRadix + d];
        g_hist[p * kRadix + d] = 0;  // self-cleaning for the next call
        const int triv = __syncthreads_or(c == n);
        unsigned long long incl;
        WarpScan(ws[warp]).InclusiveSum(c, incl);
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        unsigned long long base = 0;
        for (int w = 0; w < warp; ++w) base += s_warp[w];
        plan->digit_offset[p][d] = base + incl - c;
        if (d == 0) s_trivial[p] = triv || n == 0;
        __syncthreads();
    }
    if (d < kMaxSlots) plan->tile_counter[d] = 0;
    if (d != 0) return;

    int na = 0;
    for (int p = 0; p < np; ++p) {
        if (s_trivial[p]) continue;
        plan->digit[na] = p;
        plan->dxor[na] = (p == np - 1) ? top_xor : 0u;
        ++na;
    }
    plan->num_active = na;
    // Buffer chain: slot s writes `out` when (na-1-s) is even, else `tmp`, so
    // the last executed slot always lands in `out`. When in == out and na is
    // odd, slot 0 cannot write `out` (it is reading it): the chain then runs
    // in -> tmp -> out -> ... -> tmp and a trailing copy moves tmp to out.
    const bool in_place = (kin == kout);
    const bool shift_chain = in_place && (na % 2 == 1);
    const void* src = kin;
    const uint32_t* vsrc = vin;
    for (int s = 0; s < na; ++s) {
        bool to_out = ((na - 1 - s) % 2) == 0;
        if (shift_chain) to_out = !to_out;
        void* dst = to_out ? kout : ktmp;
        uint32_t* vdst = to_out ? vout : vtmp;
        plan->ksrc[s] = src;
        plan->kdst[s] = dst;
        plan->vsrc[s] = vsrc;
        plan->vdst[s] = vdst;
        src = dst;
        vsrc = vdst;
    }
    plan->do_copy = 0;
    if (na == 0 && !in_place) {
        plan->do_copy = 1;
        plan->copy_ksrc = kin;
        plan->copy_vsrc = vin;
    } else if (shift_chain) {
        plan->do_copy = 1;
        plan->copy_ksrc = ktmp;
        plan->copy_vsrc = vtmp;
    }
    plan->copy_kdst = kout;
    plan->copy_vdst = vout;
}

// ---------------------------------------------------------------------------
// onesweep digit pass

template <typename U, bool VALS, int THREADS, int ITEMS>
struct OnesweepSmem {
    static constexpr int WARPS = THREADS / 32;
    static constexpr int TILE = THREADS * ITEMS;
    static constexpr size_t kWhist = (size_t)WARPS * kRadix * 4;
    static constexpr size_t kKeys = (size_t)TILE * sizeof(U);
    static constexpr size_t kVals = VALS ? (size_t)TILE * 4 : 0;
    static constexpr size_t bytes = kWhist + kKeys + kVals;
};

template <typename U, bool VALS, typename LB, int THREADS, int ITEMS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) onesweep_kernel(RadixPlan* __restrict__ plan, int slot,
                                                           uint64_t n, uint32_t ntiles,
                                                           LB* __restrict__ lb_cur,
                                                           LB* __restrict__ lb_next) {
    using SM = OnesweepSmem<U, VALS, THREADS, ITEMS>;
    using W = LookbackWord<LB>;
    constexpr int WARPS = SM::WARPS;
    constexpr int TILE = SM::TILE;
    constexpr int WSEG = 32 * ITEMS;
    static_assert(THREADS >= kRadix, "one thread per digit is required");
    static_assert(TILE <= 65536, "tile ranks are kept in 16 bits");

    if (slot >= plan->num_active) return;

    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* s_whist = reinterpret_cast<uint32_t*>(smem);
    U* s_keys = reinterpret_cast<U*>(smem + SM::kWhist);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem + SM::kWhist + SM::kKeys);
    __shared__ unsigned long long s_gbase[kRadix];
    __shared__ uint32_t s_start[kRadix];
    __shared__ uint32_t s_wsum[kRadix / 32];
    __shared__ uint32_t s_tile;

    const int digit_pos = plan->digit[slot];
    const int shift = 8 * digit_pos;
    const uint32_t dxor = plan->dxor[slot];
    const U* __restrict__ src = static_cast<const U*>(plan->ksrc[slot]);
    U* __restrict__ dst = static_cast<U*>(plan->kdst[slot]);
    const uint32_t* __restrict__ vsrc = plan->vsrc[slot];
    uint32_t* __restrict__ vdst = plan->vdst[slot];
    const unsigned long long* __restrict__ goff = plan->digit_offset[digit_pos];

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const uint32_t lanemask_lt = (1u << lane) - 1u;
    uint32_t* wh = s_whist + warp * kRadix;

    for (;;) {
        if (tid == 0) s_tile = atomicAdd(&plan->tile_counter[slot], 1u);
#pragma unroll
        for (int i = lane; i < kRadix; i += 32) wh[i] = 0;
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) break;
        const uint64_t tile_base = (uint64_t)tile * TILE;
        const uint64_t rem = n - tile_base;
        const uint32_t tile_valid = rem < (uint64_t)TILE ? (uint32_t)rem : (uint32_t)TILE;
        if (lb_next != nullptr && tid < kRadix) lb_next[(size_t)tile * kRadix + tid] = 0;

        // ---- load: warp w owns keys [w*WSEG, (w+1)*WSEG) of the tile,
        // item j of lane l is key j*32+l (coalesced, and in-warp order == input order)
        U keys[ITEMS];
        uint32_t vals[VALS ? ITEMS : 1];
        const uint32_t wbase = warp * WSEG;
        if (tile_valid == TILE) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) keys[j] = __ldcs(src + tile_base + wbase + j * 32 + lane);
            if constexpr (VALS) {
#pragma unroll
                for (int j = 0; j < ITEMS; ++j)
                    vals[j] = __ldcs(vsrc + tile_base + wbase + j * 32 + lane);
            }
        } else {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                const uint32_t idx = wbase + j * 32 + lane;
                keys[j] = idx < tile_valid ? src[tile_base + idx] : U(0);
                if constexpr (VALS) vals[j] = idx < tile_valid ? vsrc[tile_base + idx] : 0u;
            }
        }

        // ---- warp-private ranking: peers with the same digit via match_any,
        // the highest peer bumps the warp's counter for that digit
        uint16_t rank[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t idx = wbase + j * 32 + lane;
            const bool valid = idx < tile_valid;
            const uint32_t d = valid ? digit_of(keys[j], shift, dxor) : (uint32_t)kRadix;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const int leader = 31 - __clz(peers);
            uint32_t old = 0;
            if (valid && lane == leader) {
                old = wh[d];
                wh[d] = old + __popc(peers);
            }
            old = __shfl_sync(0xffffffffu, old, leader);
            rank[j] = (uint16_t)(old + __popc(peers & lanemask_lt));
            __syncwarp();
        }
        __syncthreads();

        // ---- per digit: exclusive prefix over warps, tile count, publish
        uint32_t count = 0;
        if (tid < kRadix) {
#pragma unroll 4
            for (int w = 0; w < WARPS; ++w) {
                const uint32_t c = s_whist[w * kRadix + tid];
                s_whist[w * kRadix + tid] = count;
                count += c;
            }
            LB* slotp = lb_cur + (size_t)tile * kRadix + tid;
            st_relaxed(slotp, (tile == 0 ? W::kInc : W::kAgg) | (LB)count);
            // exclusive scan of the 256 tile counts (8 warps)
            uint32_t incl = count;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) s_wsum[warp] = incl;
            s_start[tid] = incl - count;  // partial (within warp)
        }
        __syncthreads();
        if (tid < kRadix) {
            uint32_t base = 0;
#pragma unroll
            for (int w = 0; w < kRadix / 32; ++w) base += (w < warp) ? s_wsum[w] : 0u;
            const uint32_t start = s_start[tid] + base;
            s_start[tid] = start;
#pragma unroll 4
            for (int w = 0; w < WARPS; ++w) s_whist[w * kRadix + tid] += start;
        }
        __syncthreads();

        // ---- stage the tile digit-sorted in shared memory
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t idx = wbase + j * 32 + lane;
            if (idx < tile_valid) {
                const uint32_t d = digit_of(keys[j], shift, dxor);
                const uint32_t r = rank[j] + wh[d];
                s_keys[r] = keys[j];
                if constexpr (VALS) s_vals[r] = vals[j];
            }
        }

        // ---- decoupled look-back: one thread per digit
        if (tid < kRadix) {
            unsigned long long excl = 0;
            if (tile > 0) {
                int64_t pred = (int64_t)tile - 1;
                const LB* col = lb_cur + tid;
                for (;;) {
                    const LB w = ld_relaxed(col + (size_t)pred * kRadix);
                    const LB f = W::flag(w);
                    if (f == 0) continue;
                    excl += (unsigned long long)(w & W::kMask);
                    if (f == 2) break;
                    --pred;
                }
                st_relaxed(lb_cur + (size_t)tile * kRadix + tid, W::kInc | (LB)(excl + count));
            }
            s_gbase[tid] = goff[tid] + excl - s_start[tid];
        }
        __syncthreads();

        // ---- write runs of equal digits: consecutive threads, consecutive slots
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t i = j * THREADS + tid;
            if (i < tile_valid) {
                const U k = s_keys[i];
                const unsigned long long g = s_gbase[digit_of(k, shift, dxor)] + i;
                dst[g] = k;
                if constexpr (VALS) vdst[g] = s_vals[i];
            }
        }
        __syncthreads();
    }
}

template <typename U>
__global__ void radix_copy_kernel(const RadixPlan* __restrict__ plan, uint64_t n, int with_vals) {
    if (!plan->do_copy) return;
    const U* __restrict__ s = static_cast<const U*>(plan->copy_ksrc);
    U* __restrict__ d = static_cast<U*>(plan->copy_kdst);
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = tid; i < n; i += stride) d[i] = s[i];
    if (with_vals) {
        const uint32_t* __restrict__ vs = plan->copy_vsrc;
        uint32_t* __restrict__ vd = plan->copy_vdst;
        for (uint64_t i = tid; i < n; i += stride) vd[i] = vs[i];
    }
}

// Tile configurations. Registers must stay <= 65536 / (THREADS * MINB) so
// MINB CTAs are resident per SM; B2S_ONESWEEP_CFG selects one for tuning runs.
struct TileCfg {
    int threads, items;
};

int onesweep_cfg() {
    static int cfg = -1;
    if (cfg < 0) {
        const char* e = getenv("B2S_ONESWEEP_CFG");
        cfg = e ? atoi(e) : 0;
    }
    return cfg;
}

template <typename U, bool VALS, typename LB, int THREADS, int ITEMS, int MINB>
b2s_status launch_passes_cfg(b2s_ctx* ctx, RadixPlan* plan, uint64_t n, void* lb) {
    using SM = OnesweepSmem<U, VALS, THREADS, ITEMS>;
    constexpr int TILE = SM::TILE;
    auto kern = onesweep_kernel<U, VALS, LB, THREADS, ITEMS, MINB>;
    static int occ = -1;  // per instantiation, per process (single device type)
    if (occ < 0) {
        B2S_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)SM::bytes));
        int o = 0;
        B2S_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, THREADS, SM::bytes));
        occ = o > 0 ? o : 1;
    }
    const uint64_t ntiles64 = (n + TILE - 1) / TILE;
    const uint32_t ntiles = (uint32_t)ntiles64;
    const uint32_t grid = (uint32_t)std::min<uint64_t>(ntiles64, (uint64_t)occ * ctx->num_sms);
    LB* region[2] = {static_cast<LB*>(lb), static_cast<LB*>(lb) + (size_t)ntiles * kRadix};
    const int slots = (int)sizeof(U);
    for (int s = 0; s < slots; ++s) {
        ctx->ev_pass[s] = record(ctx);
        kern<<<grid, THREADS, SM::bytes, ctx->stream>>>(plan, s, n, ntiles, region[s & 1],
                                                      region[(s + 1) & 1]);
        B2S_LAUNCHED();
    }
    ctx->ev_pass[slots] = record(ctx);
    return B2S_OK;
}

// smallest tile over all configurations: sizes the look-back scratch
constexpr int kMinTile = 256 * 12;

template <typename U, bool VALS, typename LB>
b2s_status launch_passes(b2s_ctx* ctx, RadixPlan* plan, uint64_t n, void* lb) {
    const int cfg = onesweep_cfg();
    if constexpr (sizeof(U) == 4) {
        if (cfg == 1) return launch_passes_cfg<U, VALS, LB, 256, 16, 4>(ctx, plan, n, lb);
        if (cfg == 2) return launch_passes_cfg<U, VALS, LB, 512, 12, 2>(ctx, plan, n, lb);
        if (cfg == 3) return launch_passes_cfg<U, VALS, LB, 384, 16, 2>(ctx, plan, n, lb);
        return launch_passes_cfg<U, VALS, LB, 512, 16, 2>(ctx, plan, n, lb);
    } else {
        if (cfg == 1) return launch_passes_cfg<U, VALS, LB, 256, 12, 4>(ctx, plan, n, lb);
        return launch_passes_cfg<U, VALS, LB, 512, 12, 2>(ctx, plan, n, lb);
    }
}

template <typename U, bool VALS>
b2s_status radix_sort_t(b2s_ctx* ctx, bool is_signed, const void* kin, void* kout,
                        const uint32_t* vin, uint32_t* vout, uint64_t n) {
    constexpr int TILE = kMinTile;
    constexpr int NP = sizeof(U);
    const uint32_t top_xor = is_signed ? 0x80u : 0u;
    const uint64_t ntiles = (n + TILE - 1) / TILE;
    const bool wide = n >= (1ull << 30);
    const size_t lb_word = wide ? 8 : 4;
    const size_t lb_region = ntiles * kRadix * lb_word;

    B2S_TRY(ctx->alt_keys.ensure(n * sizeof(U)));
    if (VALS) B2S_TRY(ctx->alt_vals.ensure(n * 4));
    B2S_TRY(ctx->lookback.ensure(2 * lb_region + 16));
    B2S_TRY(ctx->plan.ensure(sizeof(RadixPlan)));
    RadixPlan* plan = static_cast<RadixPlan*>(ctx->plan.ptr);
    unsigned long long* hist = static_cast<unsigned long long*>(ctx->hist.ptr);

    ctx->ev_hist0 = record(ctx);
    {
        const int threads = 512;
        uint64_t want = (n / (16 / sizeof(U)) + threads - 1) / threads;
        int grid = (int)std::min<uint64_t>(std::max<uint64_t>(want, 1), (uint64_t)ctx->num_sms * 4);
        radix_hist_kernel<U><<<grid, threads, 0, ctx->stream>>>(
            static_cast<const U*>(kin), n, top_xor, hist, static_cast<uint4*>(ctx->lookback.ptr),
            (lb_region + 15) / 16);
        B2S_LAUNCHED();
    }
    radix_plan_kernel<<<1, 256, 0, ctx->stream>>>(plan, hist, NP, n, top_xor, kin, kout,
                                                  ctx->alt_keys.ptr, vin, vout,
                                                  static_cast<uint32_t*>(ctx->alt_vals.ptr));
    B2S_LAUNCHED();
    ctx->ev_hist1 = record(ctx);
    ctx->last_passes_possible = NP;

    if (n > 0) {
        if (wide)
            B2S_TRY((launch_passes<U, VALS, unsigned long long>(ctx, plan, n, ctx->lookback.ptr)));
        else
            B2S_TRY((launch_passes<U, VALS, uint32_t>(ctx, plan, n, ctx->lookback.ptr)));
    }
    {
        int grid = (int)std::min<uint64_t>(std::max<uint64_t>((n + 1023) / 1024, 1),
                                           (uint64_t)ctx->num_sms * 8);
        radix_copy_kernel<U><<<grid, 256, 0, ctx->stream>>>(plan, n, VALS ? 1 : 0);
        B2S_LAUNCHED();
    }
    ctx->ev_copy1 = record(ctx);
    return B2S_OK;
}

}  // namespace

b2s_status radix_sort(b2s_ctx* ctx, b2s_dtype dtype, const void* kin, void* kout,
                      const uint32_t* vin, uint32_t* vout, uint64_t n) {
    B2S_TRY(ctx->hist.ensure(kMaxSlots * kRadix * sizeof(unsigned long long)));
    const bool sgn = key_signed(dtype);
    const bool vals = vin != nullptr;
    if (key_bytes(dtype) == 4) {
        return vals ? radix_sort_t<uint32_t, true>(ctx, sgn, kin, kout, vin, vout, n)
                    : radix_sort_t<uint32_t, false>(ctx, sgn, kin, kout, vin, vout, n);
    }
    return vals ? radix_sort_t<unsigned long long, true>(ctx, sgn, kin, kout, vin, vout, n)
                : radix_sort_t<unsigned long long, false>(ctx, sgn, kin, kout, vin, vout, n);
}

}  // namespace b2s
