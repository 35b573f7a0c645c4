// radix_sort.cu -- LSD onesweep radix sort for sm_100a.
//
// Replaces the reference's per-rank comparison sorts (kernels::merge_sort /
// quick_sort / bubble_sort, P/src/sort_core.cpp:23-144, reached through
// KernelFn, P/src/parallel_sort.cpp:136-164). The output is the same ascending
// array std::sort gives (P/src/bench.cpp:95-104); with a payload the sort is
// stable (equal keys keep input order, merge_sort's tie rule :77).
//
// Structure (one call, all on one stream, no host round trip):
//   radix_prologue_all_kernel / radix_prologue_kernel
//                          one read of the keys: OR / OR-of-complement of all
//                          keys (which bits vary, hence which 8-bit digits are
//                          constant and can be skipped), every digit's
//                          histogram (4-byte keys; 8-byte keys: digit 0), a
//                          sample of adjacent-pair order (structured input);
//                          zeroes look-back region 0 when the first pass
//                          uses it.
//   radix_order_check_kernel  when the prologue's sample of adjacent pairs is
//                          all one way (and some bit varies): counts every
//                          adjacent pair k[i] > k[i+1] and k[i] < k[i+1]; an
//                          ascending input then runs no pass at all (copied
//                          if out of place), a descending one is reversed
//                          (keys only: non-increasing; with a payload:
//                          strictly decreasing, so the order stays stable).
//                          Exits at once otherwise.
//   radix_plan_kernel      1 thread: active digit list, histogram source per
//                          slot, ping-pong buffer chain so the last executed
//                          pass lands in the output.
//   radix_fallback_hist    recounts the first active digit when the prologue
//                          did not count it (exits at once otherwise).
//   onesweep_kernel x S    per digit slot, three kernels of which one runs it
//                          (regular / skewed-pass / structured-input twins):
//                          persistent CTAs scan the slot's histogram into
//                          global digit offsets, take tiles from an atomic
//                          counter (the next one streams in by TMA), rank keys
//                          in-warp with lane-ordered shared atomics (ballot
//                          matching where the device probe fails), publish
//                          per-digit tile counts, resolve the tile's global
//                          offsets by decoupled look-back (a keys-only sort's
//                          first pass: fetch-and-add), stage the tile
//                          digit-sorted in shared memory and write runs of
//                          equal digits with coalesced stores; 8-byte keys
//                          count the NEXT slot's digit on the way out.
//   radix_copy_kernel      only does work when an in-place sort executed an
//                          odd number of passes (or zero passes out of place).
//   topfirst_fixup_kernel  8-byte keys, 2^22..2^31 of them, whose upper half
//                          varies in enough bits: only the four upper digits
//                          are sorted (stable), which leaves ties of the upper
//                          half -- a few percent of the keys, in runs of two or
//                          three -- in input order; this kernel orders every
//                          such run by its lower half (stable). A run it
//                          cannot handle raises a flag and a second, full sort
//                          (whose kernels all exit at once otherwise) follows.
//
// HBM traffic per executed pass: read + write of every key (and payload):
// 2 * (key_bytes + val_bytes) * n. The prologue reads key_bytes * n once.
#include <stdio.h>
#include <stdlib.h>

#include <string>

#include "b2s_internal.cuh"

#ifdef B2S_PHASE_PROFILE
// Debug build only (make prof): per-phase SM cycles of the onesweep kernel,
// summed over CTAs, for thread 0 (a look-back warp) and the last thread.
__device__ unsigned long long b2s_phase_cycles[2][8];
#define B2S_PHASE(k)                                                   \
    do {                                                               \
        const long long t_ = clock64();                                \
        prof_acc[k] += (unsigned long long)(t_ - prof_t);              \
        prof_t = t_;                                                   \
    } while (0)
#else
#define B2S_PHASE(k) \
    do {             \
    } while (0)
#endif

namespace b2s {
namespace {

constexpr int kRadix = 256;

// items per thread of the 4-byte-key tile (512 threads) from 2^21 keys on
#ifndef B2S_U32_ITEMS
#define B2S_U32_ITEMS 24
#endif
#ifndef B2S_U32_THREADS
#define B2S_U32_THREADS 512
#endif
#ifndef B2S_U32_MINB
#define B2S_U32_MINB 2  // CTAs per SM of that tile
#endif

#ifndef B2S_LB_PRE
// predecessors' words prefetched (cp.async) before the ranking. Round 1: 2:
// 0.719 ms per 2^28 u32 pass, 4: 0.723, 8: 0.98 (smem). With the current
// kernel only 1.5% of the look-backs finish from the prefetched words (the
// predecessors have not published yet), and none is better: 0: 0.673 ms,
// 1: 0.676, 2: 0.681 (cfg3 22.56 -> 22.25 ms, cfg5's passes 1.855 -> 1.818)
#define B2S_LB_PRE 0
#endif

// kPrefetch: predecessors whose words are prefetched before the ranking. The
// 64-bit words (n > 2^31, see narrow_lookback_words) prefetch at most one: two
// would push the static shared memory past the two-CTAs-per-SM budget
// (measured in round 1 with 2^31 i32: 7.8 ms per pass at one CTA/SM).
template <typename LB>
struct LookbackWord;
template <>
struct LookbackWord<uint32_t> {
    static constexpr uint32_t kAgg = 1u << 30, kInc = 2u << 30, kMask = (1u << 30) - 1;
    static constexpr int kPrefetch = B2S_LB_PRE;
    static __device__ __forceinline__ uint32_t flag(uint32_t w) { return w >> 30; }
};
template <>
struct LookbackWord<unsigned long long> {
    static constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62,
                                        kMask = (1ull << 62) - 1;
    static constexpr int kPrefetch = B2S_LB_PRE ? 1 : 0;
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
    // digits are whole bytes: one byte-permute extracts one (PRMT) instead of
    // a shift and a mask on the saturated ALU pipe
    uint32_t w;
    if constexpr (sizeof(U) == 4) w = (uint32_t)k;
    else w = shift >= 32 ? (uint32_t)((unsigned long long)k >> 32) : (uint32_t)k;
    return __byte_perm(w, 0u, 0x4440u | ((shift >> 3) & 3)) ^ dxor;
}

// ---------------------------------------------------------------------------
// prologue: varying-bit statistics + digit-0 histogram (one read of the keys)

// order statistic of the adjacent pairs inside one vector (the prologue
// samples one vector in four): structured input is almost all one direction
template <typename U, int D>
__device__ __forceinline__ void order_pairs(const U (&e)[D], uint32_t& asc, uint32_t& desc) {
#pragma unroll
    for (int j = 0; j + 1 < D; ++j) {
        asc += e[j] < e[j + 1];
        desc += e[j + 1] < e[j];
    }
}

template <typename U, int D, bool D4 = false>
__device__ __forceinline__ void prologue_keys(const U (&e)[D], unsigned long long& o,
                                              unsigned long long& no, uint32_t hbase) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
        o |= (unsigned long long)e[j];
        no |= (unsigned long long)(U)~e[j];
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hbase + 4u * ((uint32_t)e[j] & 0xFFu))
                     : "memory");
        if constexpr (D4 && sizeof(U) == 8) {
            // digit 4 (bits 32..39) into the second histogram, 1 KB further
            const uint32_t d4 = (uint32_t)((unsigned long long)e[j] >> 32) & 0xFFu;
            asm volatile("red.shared.add.u32 [%0+1024], 1;" ::"r"(hbase + 4u * d4) : "memory");
        }
    }
}

// CTAs per SM of the prologue (its grid is exactly one wave of them; 32
// registers per thread for u32 keys, 40 for u64)
template <typename U>
constexpr int kPrologueMinBlocks = sizeof(U) == 4 ? 4 : 3;

template <typename U, bool D4 = false>
__global__ void __launch_bounds__(512, kPrologueMinBlocks<U>) radix_prologue_kernel(const U* __restrict__ keys, uint64_t n,
                                                             RadixCounters* __restrict__ ctr,
                                                             uint4* __restrict__ lb_zero,
                                                             uint64_t lb_zero_vecs,
                                                             const RadixPlan* __restrict__ cond) {
    constexpr int VEC = 16 / sizeof(U);
    if (cond != nullptr && cond->fix_flag == 0) return;  // the conditional full sort is not needed
    __shared__ uint32_t s_h[D4 ? 2 * kRadix : kRadix];  // digit 0 | digit 4
    __shared__ unsigned long long s_or[16], s_nor[16];
    __shared__ uint2 s_ord[16];
    for (int i = threadIdx.x; i < (D4 ? 2 : 1) * kRadix; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
    const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(s_h);
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = tid; i < lb_zero_vecs; i += stride) lb_zero[i] = make_uint4(0, 0, 0, 0);

    unsigned long long o = 0, no = 0;
    uint32_t asc = 0, desc = 0;
    const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
    uint64_t head = 0;
    if (aligned) {
        const uint4* kv = reinterpret_cast<const uint4*>(keys);
        const uint64_t nvec = n / VEC;
        uint64_t v = tid;
        for (; v + 3 * stride < nvec; v += 4 * stride) {  // 4 independent 16-B loads in flight
            uint4 q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = __ldcs(kv + v + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                prologue_keys<U, VEC, D4>(*reinterpret_cast<const U(*)[VEC]>(&q[u]), o, no, hbase);
            order_pairs<U, VEC>(*reinterpret_cast<const U(*)[VEC]>(&q[0]), asc, desc);
        }
        for (; v < nvec; v += stride) {
            uint4 q = __ldcs(kv + v);
            prologue_keys<U, VEC, D4>(*reinterpret_cast<const U(*)[VEC]>(&q), o, no, hbase);
            order_pairs<U, VEC>(*reinterpret_cast<const U(*)[VEC]>(&q), asc, desc);
        }
        head = nvec * VEC;
    }
    for (uint64_t i = head + tid; i < n; i += stride) {
        const U e[1] = {keys[i]};
        prologue_keys<U, 1, D4>(e, o, no, hbase);
    }
    // block OR-reduction, then one global atomic per block
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, off);
        no |= __shfl_xor_sync(0xffffffffu, no, off);
        asc += __shfl_xor_sync(0xffffffffu, asc, off);
        desc += __shfl_xor_sync(0xffffffffu, desc, off);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s_or[warp] = o;
        s_nor[warp] = no;
        s_ord[warp] = make_uint2(asc, desc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = asc, d = desc;
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            o |= s_or[w];
            no |= s_nor[w];
            a += s_ord[w].x;
            d += s_ord[w].y;
        }
        if (o) atomicOr(&ctr->or_all, o);
        if (no) atomicOr(&ctr->nor_all, no);
        if (a) atomicAdd(&ctr->asc_pairs, a);
        if (d) atomicAdd(&ctr->desc_pairs, d);
    }
    for (int i = threadIdx.x; i < kRadix; i += blockDim.x) {
        const uint32_t c = s_h[i];
        if (c) atomicAdd(&ctr->spec0[i], (unsigned long long)c);
        if constexpr (D4) {
            const uint32_t c4 = s_h[kRadix + i];
            if (c4) atomicAdd(&ctr->spec4[i], (unsigned long long)c4);
        }
    }
}

// All-digit prologue: every digit histogram in one read, so the passes need
// not count the next digit on their way out (that count is a random shared
// atomic per key, ~7% of a pass). Lanes own columns of counters
// (s_hl[digit][bin][column]): 4-byte keys give each lane its own column (the
// bank is the lane: the four per-key shared reductions are conflict-free);
// 8-byte keys have 8 digits, so lanes l and l+16 share one of 16 columns
// (at most 2-way conflicts) and the columns still fit 128 KB. One
// 1024-thread CTA per SM. Also the OR / OR-of-complement and the
// adjacent-pair order sample of the regular prologue.
#ifndef B2S_ALLHIST_DEPTH
#define B2S_ALLHIST_DEPTH 8  // 8: 0.227 -> 0.217 ms for 2^28 u32 (4)
#endif
constexpr int kAllHistThreads = 1024;
constexpr size_t kAllHistSmem = 128 * 1024;
constexpr uint64_t kAllHistMinKeys = 1ull << 22;

template <typename U>
__global__ void __launch_bounds__(kAllHistThreads, 1)
    radix_prologue_all_kernel(const U* __restrict__ keys, uint64_t n,
                              RadixCounters* __restrict__ ctr, uint4* __restrict__ lb_zero,
                              uint64_t lb_zero_vecs, uint32_t top_xor,
                              const RadixPlan* __restrict__ cond) {
    constexpr int ND = sizeof(U);            // digits
    if (cond != nullptr && cond->fix_flag == 0) return;
    constexpr int COLS = sizeof(U) == 4 ? 32 : 16;
    constexpr int VEC = 16 / sizeof(U);      // keys per 16-byte load
    static_assert((size_t)ND * 256 * COLS * 4 == kAllHistSmem, "column layout");
    extern __shared__ __align__(16) uint32_t s_hl[];  // [ND][256][COLS]
    __shared__ unsigned long long s_or[32], s_nor[32];
    __shared__ uint2 s_ord[32];
    for (int i = threadIdx.x; i < (int)(kAllHistSmem / 16); i += blockDim.x)
        reinterpret_cast<uint4*>(s_hl)[i] = make_uint4(0, 0, 0, 0);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t hb = (uint32_t)__cvta_generic_to_shared(s_hl) + 4u * (lane & (COLS - 1));
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = tid; i < lb_zero_vecs; i += stride) lb_zero[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    unsigned long long o = 0, no = 0;
    uint32_t asc = 0, desc = 0;
    // counter of (digit p, bin b) in this lane's column: hb + (p*256 + b)*COLS*4
    auto count = [&](U e) {
        o |= (unsigned long long)e;
        no |= (unsigned long long)(U)~e;
        if constexpr (sizeof(U) == 4) {
            const uint32_t tx7 = top_xor << 7;
            const uint32_t a0 = ((uint32_t)e << 7) & 0x7F80u;
            const uint32_t a1 = ((uint32_t)e >> 1) & 0x7F80u;
            const uint32_t a2 = ((uint32_t)e >> 9) & 0x7F80u;
            const uint32_t a3 = (((uint32_t)e >> 17) & 0x7F80u) ^ tx7;
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hb + a0) : "memory");
            asm volatile("red.shared.add.u32 [%0+32768], 1;" ::"r"(hb + a1) : "memory");
            asm volatile("red.shared.add.u32 [%0+65536], 1;" ::"r"(hb + a2) : "memory");
            asm volatile("red.shared.add.u32 [%0+98304], 1;" ::"r"(hb + a3) : "memory");
        } else {
            const uint32_t lo = (uint32_t)e, hi = (uint32_t)((unsigned long long)e >> 32);
            const uint32_t tx6 = top_xor << 6;
            // bin * 64 bytes: byte k of a word at bits 6..13
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hb + ((lo << 6) & 0x3FC0u)) : "memory");
            asm volatile("red.shared.add.u32 [%0+16384], 1;" ::"r"(hb + ((lo >> 2) & 0x3FC0u)) : "memory");
            asm volatile("red.shared.add.u32 [%0+32768], 1;" ::"r"(hb + ((lo >> 10) & 0x3FC0u)) : "memory");
            asm volatile("red.shared.add.u32 [%0+49152], 1;" ::"r"(hb + ((lo >> 18) & 0x3FC0u)) : "memory");
            asm volatile("red.shared.add.u32 [%0+65536], 1;" ::"r"(hb + ((hi << 6) & 0x3FC0u)) : "memory");
            asm volatile("red.shared.add.u32 [%0+81920], 1;" ::"r"(hb + ((hi >> 2) & 0x3FC0u)) : "memory");
            asm volatile("red.shared.add.u32 [%0+98304], 1;" ::"r"(hb + ((hi >> 10) & 0x3FC0u)) : "memory");
            asm volatile("red.shared.add.u32 [%0+114688], 1;" ::"r"(hb + (((hi >> 18) & 0x3FC0u) ^ tx6))
                         : "memory");
        }
    };
    const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
    uint64_t head = 0;
    if (aligned) {
        const uint4* kv = reinterpret_cast<const uint4*>(keys);
        const uint64_t nvec = n / VEC;
        uint64_t v = tid;
        constexpr int QD = B2S_ALLHIST_DEPTH;  // independent 16-B loads in flight per thread
        for (; v + (QD - 1) * stride < nvec; v += QD * stride) {
            uint4 q[QD];
#pragma unroll
            for (int u = 0; u < QD; ++u) q[u] = __ldcs(kv + v + u * stride);
#pragma unroll
            for (int u = 0; u < QD; ++u) {
                const U(&e)[VEC] = *reinterpret_cast<const U(*)[VEC]>(&q[u]);
#pragma unroll
                for (int j = 0; j < VEC; ++j) count(e[j]);
            }
            order_pairs<U, VEC>(*reinterpret_cast<const U(*)[VEC]>(&q[0]), asc, desc);
        }
        for (; v < nvec; v += stride) {
            const uint4 q = __ldcs(kv + v);
            const U(&e)[VEC] = *reinterpret_cast<const U(*)[VEC]>(&q);
#pragma unroll
            for (int j = 0; j < VEC; ++j) count(e[j]);
            order_pairs<U, VEC>(e, asc, desc);
        }
        head = nvec * VEC;
    }
    for (uint64_t i = head + tid; i < n; i += stride) count(keys[i]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, off);
        no |= __shfl_xor_sync(0xffffffffu, no, off);
        asc += __shfl_xor_sync(0xffffffffu, asc, off);
        desc += __shfl_xor_sync(0xffffffffu, desc, off);
    }
    const int warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_or[warp] = o;
        s_nor[warp] = no;
        s_ord[warp] = make_uint2(asc, desc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, d = 0;
        o = 0;
        no = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            o |= s_or[w];
            no |= s_nor[w];
            a += s_ord[w].x;
            d += s_ord[w].y;
        }
        if (o) atomicOr(&ctr->or_all, o);
        if (no) atomicOr(&ctr->nor_all, no);
        if (a) atomicAdd(&ctr->asc_pairs, a);
        if (d) atomicAdd(&ctr->desc_pairs, d);
    }
    // column sums: thread i sums row i starting at column i (spread banks)
    for (int i = threadIdx.x; i < ND * 256; i += blockDim.x) {
        const uint32_t* row = s_hl + i * COLS;
        uint32_t sum = 0;
#pragma unroll 8
        for (int l = 0; l < COLS; ++l) sum += row[(l + i) & (COLS - 1)];
        if (sum) atomicAdd(&ctr->dhist[i >> 8][i & 255], (unsigned long long)sum);
    }
}

// ---------------------------------------------------------------------------
// exact order check of presorted-looking input
constexpr uint64_t kOrderCheckMinKeys = 1ull << 20;

template <typename U>
__global__ void __launch_bounds__(512) radix_order_check_kernel(const U* __restrict__ keys, uint64_t n,
                                                                 RadixCounters* __restrict__ ctr,
                                                                 U flip) {
    // gate: the sampled pairs (raw unsigned compare; a signed array crossing
    // zero shows one odd pair) are all one way, and the keys are not all equal
    {
        const unsigned long long a = ctr->asc_pairs, d = ctr->desc_pairs;
        if ((a < d ? a : d) > 2 || (ctr->or_all & ctr->nor_all) == 0) return;
    }
    constexpr int VEC = 16 / sizeof(U);
    const int lane = threadIdx.x & 31;
    unsigned long long gt = 0, lt = 0;
    auto cmp = [&](U x, U y) {  // x before y in the input
        x ^= flip;
        y ^= flip;
        gt += x > y;
        lt += x < y;
    };
    if ((reinterpret_cast<uintptr_t>(keys) & 15) == 0) {
        const uint4* kv = reinterpret_cast<const uint4*>(keys);
        const uint64_t nvec = n / VEC;
        const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
        const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
        for (uint64_t v0 = warp * 32; v0 < nvec; v0 += nwarps * 32) {  // warp-uniform trips
            const uint64_t v = v0 + lane;
            uint4 q = make_uint4(0, 0, 0, 0);
            if (v < nvec) q = __ldcs(kv + v);
            const U(&e)[VEC] = *reinterpret_cast<const U(*)[VEC]>(&q);
            // the next vector's first element: the next lane's, or one load
            U nxt;
            if constexpr (sizeof(U) == 4) {
                nxt = (U)__shfl_down_sync(0xffffffffu, (uint32_t)e[0], 1);
            } else {
                nxt = (U)__shfl_down_sync(0xffffffffu, (unsigned long long)e[0], 1);
            }
            if (v < nvec) {
#pragma unroll
                for (int j = 0; j + 1 < VEC; ++j) cmp(e[j], e[j + 1]);
                const uint64_t ni = (v + 1) * VEC;
                if (ni < n) cmp(e[VEC - 1], (lane < 31 && v + 1 < nvec) ? nxt : keys[ni]);
            }
        }
        // the tail after the last whole vector
        if (blockIdx.x == 0 && threadIdx.x == 0)
            for (uint64_t i = nvec * VEC; i + 1 < n; ++i) cmp(keys[i], keys[i + 1]);
    } else {
        const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += stride)
            cmp(keys[i], keys[i + 1]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        gt += __shfl_xor_sync(0xffffffffu, gt, off);
        lt += __shfl_xor_sync(0xffffffffu, lt, off);
    }
    if (lane == 0) {
        if (gt) atomicAdd(&ctr->gt_pairs, gt);
        if (lt) atomicAdd(&ctr->lt_pairs, lt);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->order_checked = 1;
}

// ---------------------------------------------------------------------------
// pass plan: active digits, histogram per slot, buffer chain

__global__ void radix_plan_kernel(RadixPlan* __restrict__ plan, RadixCounters* __restrict__ ctr,
                                  int np, uint64_t n, uint32_t top_xor, const void* kin,
                                  void* kout, void* ktmp, const uint32_t* vin, uint32_t* vout,
                                  uint32_t* vtmp, int all_hist, int top_mode,
                                  const RadixPlan* __restrict__ cond) {
    if (threadIdx.x < kMaxSlots) plan->tile_counter[threadIdx.x] = 0;
    if (threadIdx.x != 0) return;
    plan->topfirst = 0;
    plan->fix_flag = 0;
    if (top_mode == 2 && cond->fix_flag == 0) {  // the fix-up finished the sort: nothing to do
        plan->num_active = 0;
        plan->do_copy = 0;
        plan->need_fallback = 0;
        plan->structured = 0;
        plan->all_hist = 0;
        return;
    }
    // a bit varies iff some key has it set and some key has it clear
    const unsigned long long varying = ctr->or_all & ctr->nor_all;
    // Upper-digits-first (top_mode 1, 8-byte keys): with b varying bits in the
    // upper half, n keys fall into ~2^b classes of equal upper halves; from
    // b >= log2(n) + 2 on at most ~1/8 of the keys share their class, in runs
    // of two or three, which the fix-up kernel orders. The four lower passes
    // are then not run at all.
    unsigned int dmask = 0xFFu;
    if (top_mode == 1) {
        const int hi_bits = __popcll(varying >> 32), lo_bits = __popcll(varying & 0xFFFFFFFFull);
        int need = 2;
        while (need - 2 < 62 && (1ull << (need - 2)) < n) ++need;  // ceil(log2 n) + 2
        // and digit 4 must not be concentrated (a few distinct upper halves
        // can vary in every bit): no bin above n / 32 (uniform keys: n / 256)
        unsigned long long max4 = 0;
        for (int b = 0; b < 256; ++b) max4 = ctr->spec4[b] > max4 ? ctr->spec4[b] : max4;
        if (lo_bits > 0 && hi_bits >= (need < 32 ? need : 32) && !all_hist && max4 <= n / 32) {
            dmask = 0xF0u;
            plan->topfirst = 1;
        }
    }
    int na = 0;
    for (int p = 0; p < np && n > 0; ++p) {
        if (((varying >> (8 * p)) & 0xFFull) == 0) continue;  // constant digit: identity pass
        if (((dmask >> p) & 1u) == 0) continue;               // left to the fix-up
        plan->digit[na] = p;
        plan->dxor[na] = (p == np - 1) ? top_xor : 0u;
        plan->hist[na] = all_hist ? ctr->dhist[p] : ctr->hist[na];
        ++na;
    }
    // presorted input (radix_order_check_kernel counted every adjacent pair):
    // ascending runs no pass; descending (with a payload: strictly) is reversed
    bool reversed = false;
    if (top_mode != 2 && ctr->order_checked && n > 1) {
        const unsigned long long gt = ctr->gt_pairs, lt = ctr->lt_pairs;
        if (gt == 0) {
            na = 0;
        } else if (vin != nullptr ? gt == n - 1 : lt == 0) {
            na = 0;
            reversed = true;
        }
        if (na == 0) plan->topfirst = 0;
    }
    plan->num_active = na;
    // structured input (sorted, reverse, nearly so): adjacent pairs almost all
    // in one direction. Its passes scatter with strided slots, so they run
    // the bank-swizzled kernel.
    {
        const unsigned long long a = ctr->asc_pairs, d = ctr->desc_pairs;
        const unsigned long long hi = a > d ? a : d, lo = a > d ? d : a;
        plan->structured = hi > 8 * lo && hi > n / 16;
    }
    plan->all_hist = all_hist;
    plan->need_fallback = !all_hist && (na > 0 && plan->digit[0] != 0);
    if (!all_hist && na > 0 && plan->digit[0] == 0) plan->hist[0] = ctr->spec0;
    if (!all_hist && top_mode == 1 && na > 0 && plan->digit[0] == 4) {  // counted by the prologue too
        plan->hist[0] = ctr->spec4;
        plan->need_fallback = 0;
    }
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
    if (reversed) {
        plan->do_copy = 2;
        plan->copy_ksrc = kin;
        plan->copy_vsrc = vin;
    } else if (na == 0 && !in_place) {
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

// Histogram of the first active digit when it is not digit 0.
template <typename U>
__global__ void __launch_bounds__(512) radix_fallback_hist_kernel(const RadixPlan* __restrict__ plan,
                                                                  const U* __restrict__ keys,
                                                                  uint64_t n,
                                                                  RadixCounters* __restrict__ ctr) {
    if (!plan->need_fallback) return;
    __shared__ uint32_t s_h[kRadix];
    for (int i = threadIdx.x; i < kRadix; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
    const int shift = 8 * plan->digit[0];
    const uint32_t dxor = plan->dxor[0];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        atomicAdd(&s_h[digit_of(keys[i], shift, dxor)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < kRadix; i += blockDim.x)
        if (s_h[i]) atomicAdd(&ctr->hist[0][i], (unsigned long long)s_h[i]);
}

// ---------------------------------------------------------------------------
// onesweep digit pass
#ifndef B2S_MATCH_HYBRID
#define B2S_MATCH_HYBRID 2
#endif
constexpr bool MATCH_SMEM = B2S_MATCH_HYBRID != 0;
#ifndef B2S_ERANK
#define B2S_ERANK 1
#endif
#ifndef B2S_SEP
#define B2S_SEP 1
#endif
#ifndef B2S_ARITH_MIN_RANK
#define B2S_ARITH_MIN_RANK 3  // 2 (regular kernel too): 0.750 vs 0.720 ms per 2^28 u32 pass
#endif
// predecessors read per look-back step. With the paired walk (two digits per
// lane, 64-bit loads): 4: 0.667 ms per 2^28 u32 pass, 6: 0.664, 8: 0.667,
// 12: 0.677 (cfg3 22.00 -> 21.95 ms with 6)
#ifndef B2S_LB_STEP
#define B2S_LB_STEP 6
#endif
// 32-bit look-back words: one lane walks two adjacent digits, reading and
// publishing their two words as one 64-bit access (both always carry the same
// flag), so four warps poll instead of eight.
#ifndef B2S_LB_PAIR
#define B2S_LB_PAIR 1
#endif
#ifndef B2S_LB_WARP0
// first of the four paired look-back warps: not the four scanning warps
// (0-3), which already carry the digit section (per 2^28 u32 pass, uniform /
// ascending-but-one-pair: warp 0: 0.669 / 0.613 ms, 4: 0.667 / 0.599, 8 and
// 12 the same as 4)
#define B2S_LB_WARP0 4
#endif
#ifndef B2S_LB_SKIP_EMPTY
#define B2S_LB_SKIP_EMPTY 1
#endif
#ifndef B2S_TICKET_FIRST
#define B2S_TICKET_FIRST 1  // keys-only first pass: offsets by fetch-and-add, no look-back
#endif
#ifndef B2S_TMA_EVICT_FIRST
#define B2S_TMA_EVICT_FIRST 1
#endif
#ifndef B2S_STORE_PLAIN
#define B2S_STORE_PLAIN 0
#endif
#ifndef B2S_EARLY_LB
#define B2S_EARLY_LB 0
#endif
#ifndef B2S_ECNT_IN_CNT
#define B2S_ECNT_IN_CNT 1
#endif
#ifndef B2S_EARLY_CLAIM
#define B2S_EARLY_CLAIM 0  // 1: next tile streamed in after the early counts: 0.709 vs 0.699 ms per pass
#endif
#ifndef B2S_NAMED_SCAN
#define B2S_NAMED_SCAN 1
#endif
#ifndef B2S_ERANK_RELOAD
#define B2S_ERANK_RELOAD 1
#endif
//
// Shared-memory traffic is this kernel's bound on B200 (HBM is 6.5 TB/s but
// the random-access shared memory work per key is ~15-20 wavefronts per 32
// keys), so the layout minimises wavefronts: per-warp digit counters are
// packed two 16-bit counters per word (a warp-tile count is <= 8192), ranks
// are claimed by one shared atomic per digit group (the group's highest lane)
// and broadcast with a shuffle, and global offsets are 32-bit when n <= 2^31.

template <typename U, bool VALS, int THREADS, int ITEMS>
struct OnesweepSmem {
    static constexpr int WARPS = THREADS / 32;
    static constexpr int TILE = THREADS * ITEMS;
    static constexpr size_t kCnt = (size_t)WARPS * (kRadix / 2) * 4;  // packed u16 pairs
    static constexpr size_t kKeys = (size_t)TILE * sizeof(U);         // one tile buffer
    static constexpr size_t kVals = VALS ? (size_t)TILE * 4 : 0;
    // counters | keys[2] | vals[2]: tile i+1 streams in by TMA while tile i is
    // ranked in place in its own buffer. The early-rank kernels count into
    // s_cnt itself; the others keep their per-warp early counts and match
    // masks (WARPS x 1 KB) in the idle tile buffer until the next tile's copy
    // is issued (after the look-back).
    static constexpr size_t bytes = kCnt + 2 * kKeys + 2 * kVals;
    static_assert(kKeys >= (size_t)WARPS * kRadix * 4, "idle tile buffer holds the early counts");
};

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier ----------
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
#if B2S_TMA_EVICT_FIRST
    // the pass reads every key exactly once: ask L2 to evict the tile first
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n\t}"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar)
        : "memory");
#else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mbar)
        : "memory");
#endif
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cp_async_lb(uint32_t dst, const uint32_t* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_lb(uint32_t dst, const unsigned long long* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Lanes of the warp whose digit equals mine, from one ballot per digit bit
// (VOTE + logic ops only: MATCH.ANY serialises on the SM's shared ADU pipe).
template <int BITS>
__device__ __forceinline__ uint32_t match_digit(uint32_t d) {
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        uint32_t m;
        asm("{\n\t.reg .pred p;\n\t"
            "and.b32 %0, %1, %2;\n\t"
            "setp.ne.u32 p, %0, 0;\n\t"
            "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
            "@!p not.b32 %0, %0;\n\t}"
            : "=r"(m)
            : "r"(d), "r"(1u << b));
        peers &= m;
    }
    return peers;
}

// Shared-memory match: every valid lane ORs its bit into its digit's mask,
// reads the mask back (= its peers), and clears it. The warp is converged and
// its shared accesses run in program order, so all ORs land before the reads
// and all reads before the clears.
__device__ __forceinline__ uint32_t match_smem(bool valid, uint32_t a, uint32_t bit) {
    uint32_t peers;
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.u32 q, %1, 0;\n\t"
        "@q red.shared.or.b32 [%2], %3;\n\t"
        "@q ld.volatile.shared.u32 %0, [%2];\n\t"
        "@q st.volatile.shared.u32 [%2], 0;\n\t}"
        : "=r"(peers)
        : "r"((uint32_t)valid), "r"(a), "r"(bit)
        : "memory");
    return valid ? peers : 0u;
}

// 32-bit shared-window addressing, computed once per kernel
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void red_add_shared(uint32_t a, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
    return old;
}
// predicated shared atomic add returning the old word (0 when !pred)
__device__ __forceinline__ uint32_t atom_add_shared_if(bool pred, uint32_t a, uint32_t v) {
    uint32_t old = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t"
                 "@q atom.shared.add.u32 %0, [%1], %2;\n\t}"
                 : "+r"(old)
                 : "r"(a), "r"(v), "r"((uint32_t)pred)
                 : "memory");
    return old;
}
__device__ __forceinline__ void sts_key(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_key(uint32_t a, unsigned long long v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

// Bank swizzle of a staged tile slot: slot r sits at r ^ (its 128-byte row
// index mod the row's element count). Rows stay whole, so the write-out's
// consecutive reads stay conflict-free, while the ranking's scatter -- whose
// slots are strided when the input is structured (sorted input: a warp's 32
// keys go to 32 digit runs of equal length, all on 2 banks) -- spreads over
// the banks.
// It costs two ALU ops per key, so only passes over structured input (see
// radix_plan_kernel) use it.
template <int BYTES, bool SWZ>
__device__ __forceinline__ uint32_t swz(uint32_t r) {
    constexpr uint32_t EPR = 128 / BYTES;  // elements per 128-byte row
    return SWZ ? r ^ ((r / EPR) & (EPR - 1)) : r;
}

struct NextDigit {
    int shift;
    uint32_t dxor;
    bool on;
    uint32_t* hist;  // the next slot's digit counters (shared memory)
};

// Shared state of one CTA besides the tile buffers.
template <typename LB>
struct TileShared {
    using OFF = LB;  // 32-bit offsets exactly when the look-back words are 32-bit (n <= 2^31)
    OFF goff[kRadix];    // the slot's global digit offsets
    uint32_t dcount[sizeof(LB) == 4 ? kRadix : 1];  // 32-bit words: the slot's digit totals
    unsigned long long n;
    uint32_t nhist[kRadix];
    uint32_t start[kRadix];
    uint32_t wsum[kRadix / 32];
    unsigned long long wsum64[kRadix / 32];
    alignas(16) LB lbw[LookbackWord<LB>::kPrefetch > 0 ? LookbackWord<LB>::kPrefetch * kRadix : 4];  // prefetched look-back window
    uint32_t tile[2];
    uint32_t dummy[32];  // sink of the non-leaders' no-op rank atomics
    alignas(8) unsigned long long mbar[2];
};

// Decoupled look-back of one digit (thread tid < kRadix owns digit tid): the
// sum of the digit's counts over all tiles before `tile`. The first kPrefetch
// predecessors were fetched into `lbw` by cp.async before the ranking; later
// steps read B2S_LB_STEP at a time (independent loads) in a warp-uniform loop.
// The tile's inclusive prefix is published the moment it is known.
// 32-bit words hold prefixes modulo 2^30; `lo` is a lower bound of the true
// exclusive prefix less than 2^30 below it (narrow_lookback_words), which makes
// the residue exact.
template <typename LB>
__device__ __forceinline__ unsigned long long lookback_exclusive(uint32_t tile, LB* __restrict__ lb_cur,
                                                                 const LB* lbw, uint32_t mycount,
                                                                 unsigned long long lo,
                                                                 bool empty_digit = false) {
    using W = LookbackWord<LB>;
    constexpr int PRE = W::kPrefetch;
    constexpr int LOOKBACK = B2S_LB_STEP;
    const int tid = threadIdx.x;
    unsigned long long excl = 0;
    (void)lo;
    if (tile == 0) return 0;
    int64_t pred = (int64_t)tile - 1;
    // a digit no key of the pass has (its lane in every tile knows, from the
    // pass's histogram) needs no prefix: its lanes sit the walk out
    bool done = empty_digit;
    const LB* col = lb_cur + tid;
    LB* mine = lb_cur + (size_t)tile * kRadix + tid;
    asm volatile("cp.async.wait_all;" ::: "memory");
    bool stop = false;
#pragma unroll
    for (int i = 0; i < PRE; ++i) {
        if (!stop) {
            const LB w = ((int64_t)tile - 1 - i >= 0) ? lbw[i * kRadix + tid] : W::kInc;
            const LB f = W::flag(w);
            if (f != 0) {
                excl += (unsigned long long)(w & W::kMask);
                done = (f == 2);
                stop = done;
                pred -= done ? 0 : 1;
            } else {
                stop = true;
            }
        }
    }
    if (done) st_relaxed(mine, W::kInc | ((LB)(excl + mycount) & W::kMask));
    while (__any_sync(0xffffffffu, !done)) {
        if (!done) {
            LB w[LOOKBACK];
#pragma unroll
            for (int i = 0; i < LOOKBACK; ++i)
                w[i] = (pred - i >= 0) ? ld_relaxed(col + (size_t)(pred - i) * kRadix) : W::kInc;
            stop = false;
#pragma unroll
            for (int i = 0; i < LOOKBACK; ++i) {
                const LB f = W::flag(w[i]);
                if (!stop && f != 0) {
                    excl += (unsigned long long)(w[i] & W::kMask);
                    done = (f == 2);
                    stop = done;
                    pred -= done ? 0 : 1;
                } else {
                    stop = true;
                }
            }
            if (done) st_relaxed(mine, W::kInc | ((LB)(excl + mycount) & W::kMask));
        }
    }
    if constexpr (sizeof(LB) == 4) excl = lo + ((excl - lo) & W::kMask);
    return excl;
}

// The same walk for a pair of adjacent digits (32-bit words): thread t < 128
// owns digits 2t and 2t+1, whose words every tile publishes together in one
// 64-bit store -- aggregates in the digit section, inclusive prefixes here --
// so both carry the same flag and one 64-bit load serves both digits.
__device__ __forceinline__ void lookback_exclusive_pair(uint32_t tile, uint32_t* __restrict__ lb_cur,
                                                        uint32_t count0, uint32_t count1,
                                                        unsigned long long lo0, unsigned long long lo1,
                                                        bool empty_pair, unsigned long long& e0,
                                                        unsigned long long& e1) {
    using W = LookbackWord<uint32_t>;
    constexpr int LOOKBACK = B2S_LB_STEP;
    const int tid = threadIdx.x - 32 * B2S_LB_WARP0;  // pair index
    e0 = 0;
    e1 = 0;
    if (tile == 0) return;
    int64_t pred = (int64_t)tile - 1;
    bool done = empty_pair;
    uint32_t x0 = 0, x1 = 0;  // prefixes modulo 2^30 (sums of 30-bit residues wrap in 32 bits harmlessly)
    const unsigned long long* col = reinterpret_cast<const unsigned long long*>(lb_cur) + tid;
    unsigned long long* mine = reinterpret_cast<unsigned long long*>(lb_cur) + (size_t)tile * (kRadix / 2) + tid;
    auto publish = [&]() {
        const uint32_t w0 = W::kInc | ((x0 + count0) & W::kMask), w1 = W::kInc | ((x1 + count1) & W::kMask);
        st_relaxed(mine, (unsigned long long)w0 | ((unsigned long long)w1 << 32));
    };
    if (done) publish();
    while (__any_sync(0xffffffffu, !done)) {
        if (!done) {
            unsigned long long w[LOOKBACK];
#pragma unroll
            for (int i = 0; i < LOOKBACK; ++i)
                w[i] = (pred - i >= 0) ? ld_relaxed(col + (size_t)(pred - i) * (kRadix / 2))
                                       : ((unsigned long long)W::kInc | ((unsigned long long)W::kInc << 32));
            bool stop = false;
#pragma unroll
            for (int i = 0; i < LOOKBACK; ++i) {
                const uint32_t a = (uint32_t)w[i], b = (uint32_t)(w[i] >> 32);
                const uint32_t f = W::flag(a);  // == W::flag(b)
                if (!stop && f != 0) {
                    x0 += a & W::kMask;
                    x1 += b & W::kMask;
                    done = (f == 2);
                    stop = done;
                    pred -= done ? 0 : 1;
                } else {
                    stop = true;
                }
            }
            if (done) publish();
        }
    }
    e0 = lo0 + (((unsigned long long)x0 - lo0) & W::kMask);
    e1 = lo1 + (((unsigned long long)x1 - lo1) & W::kMask);
}

// Per-warp early counts of one full tile: the warp's keys are counted into
// its own packed 16-bit digit counters (`ecnt`, HALF words) and the returned
// old values are the keys' stable in-warp ranks (same-word lanes of one
// atomic are served in lane order, b2s::probe_lane_order), packed two per
// word in `rr`. HOT: the pass's hot digit is ranked by one ballot per row
// against a warp-uniform running count instead (same-address atomics
// serialise).
template <typename U, int ITEMS, bool HOT>
__device__ __forceinline__ void early_ranks(const U (&keys)[ITEMS], uint32_t (&rr)[(ITEMS + 1) / 2],
                                            uint32_t* ecnt, int shift, uint32_t dxor, uint32_t hot) {
    const int lane = threadIdx.x & 31;
    {
        uint4* z = reinterpret_cast<uint4*>(ecnt);
#pragma unroll
        for (int i = lane; i < kRadix / 8; i += 32) z[i] = make_uint4(0, 0, 0, 0);
        __syncwarp();
    }
    const uint32_t ecnt_a = smem_addr(ecnt);
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t hot_run = 0;
    constexpr int B = 4;
#pragma unroll
    for (int j0 = 0; j0 < ITEMS; j0 += B) {
        uint32_t old[B], s16[B], hr[B];
        bool h[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            if (j0 + b < ITEMS) {
                const uint32_t d = digit_of(keys[j0 + b], shift, dxor);
                s16[b] = 16 * (d & 1);
                if constexpr (HOT) {
                    h[b] = d == hot;
                    const uint32_t hm = __ballot_sync(0xffffffffu, h[b]);
                    hr[b] = hot_run + __popc(hm & lt);
                    hot_run += __popc(hm);
                    old[b] = atom_add_shared_if(!h[b], ecnt_a + 4 * (d >> 1), 1u << s16[b]);
                } else {
                    old[b] = atom_add_shared(ecnt_a + 4 * (d >> 1), 1u << s16[b]);
                }
            }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int j = j0 + b;
            if (j < ITEMS) {
                uint32_t r = (old[b] >> s16[b]) & 0xFFFFu;
                if constexpr (HOT) r = h[b] ? hr[b] : r;
                if (j & 1) rr[j >> 1] |= r << 16;
                else rr[j >> 1] = r;
            }
        }
    }
    if constexpr (HOT) {
        if (lane == 0 && hot_run) atomicAdd(ecnt + (hot >> 1), hot_run << (16 * (hot & 1)));
    }
}

// One tile: keys come from `kbuf` (landed by TMA) when FROM_SMEM, else from
// global memory; the tile is ranked, staged digit-sorted back into
// `kbuf`/`vbuf`, and written out.
// Write-out of a staged tile: runs of equal digits go to consecutive global
// slots (consecutive threads, consecutive positions); the next slot's digit is
// counted on the way out.
template <typename U, bool VALS, typename LB, int THREADS, int ITEMS, bool AGG = false,
          bool SWZ = false>
__device__ __forceinline__ void writeout_tile(const U* kbuf, const uint32_t* vbuf,
                                              const typename TileShared<LB>::OFF* gbase,
                                              uint32_t tile_valid, U* __restrict__ dst,
                                              uint32_t* __restrict__ vdst, int shift, uint32_t dxor,
                                              const NextDigit nd) {
    using OFF = typename TileShared<LB>::OFF;
    const bool full = tile_valid == (uint32_t)(THREADS * ITEMS);
    constexpr uint32_t EPR = 128 / sizeof(U);
    static_assert(THREADS % EPR == 0, "whole rows per item step");
    const uint32_t q = threadIdx.x / EPR;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const uint32_t i = j * THREADS + threadIdx.x;
        if (full || i < tile_valid) {
            // swz(i) with the row term folded: j * THREADS is a whole number
            // of rows, so only the low bits of threadIdx.x are permuted
            const uint32_t si = SWZ ? j * THREADS + (threadIdx.x ^ (((uint32_t)(j * THREADS / EPR) + q) & (EPR - 1)))
                                            : i;
            const U k = kbuf[si];
            const OFF g = gbase[digit_of(k, shift, dxor)] + (OFF)i;
            // streaming (evict-first) stores, except for structured input,
            // whose runs land in few, long stretches (measured per 2^28-key
            // u32 pass: uniform 0.718 streaming vs 0.725 plain, ascending
            // 0.668 vs 0.654)
            if constexpr (SWZ || B2S_STORE_PLAIN) {
                dst[g] = k;
                if constexpr (VALS) vdst[g] = vbuf[sizeof(U) == 4 ? si : swz<4, SWZ>(i)];
            } else {
                __stcs(dst + g, k);
                if constexpr (VALS) __stcs(vdst + g, vbuf[sizeof(U) == 4 ? si : swz<4, SWZ>(i)]);
            }
            if (nd.on) {
                const uint32_t dn = digit_of(k, nd.shift, nd.dxor);
                if (AGG && full) {
                    // skewed pass: lanes sharing lane 0's next digit count it
                    // with one add (same-address atomics serialise)
                    const uint32_t d0 = __shfl_sync(0xffffffffu, dn, 0);
                    const uint32_t m = __ballot_sync(0xffffffffu, dn == d0);
                    if (dn != d0) atomicAdd(nd.hist + dn, 1u);
                    else if ((threadIdx.x & 31) == 0) atomicAdd(nd.hist + d0, (uint32_t)__popc(m));
                } else {
                    atomicAdd(nd.hist + dn, 1u);  // ATOMS.POPC.INC
                }
            }
        }
    }
}

template <typename U, bool VALS, typename LB, int THREADS, int ITEMS, bool FULL, bool FROM_SMEM,
          int RANK, bool SWZ = false, bool SEP = false, typename Claim, typename Between>
__device__ __forceinline__ void onesweep_tile(const Claim& claim_next, const Between& between,
                                              typename TileShared<LB>::OFF* gbase_out, uint32_t tile,
                                              uint32_t tile_valid, uint64_t tile_base,
                                              const U* __restrict__ src, U* __restrict__ dst,
                                              const uint32_t* __restrict__ vsrc,
                                              uint32_t* __restrict__ vdst, LB* __restrict__ lb_cur,
                                              unsigned long long* __restrict__ ticket, int shift,
                                              uint32_t dxor, const NextDigit nd,
                                              uint32_t* s_cnt, U* kbuf, uint32_t* vbuf,
                                              U* sbuf, uint32_t* svbuf,
                                              uint32_t* s_match, uint32_t* s_early,
                                              TileShared<LB>& sh,
                                              unsigned long long* prof_acc,
                                              long long& prof_t, uint32_t hot = 0) {
    // RANK: 0 ballot matching, 1 lane-ordered atomics, 2 atomics except for
    // the pass's hot digit, whose lanes are counted and ranked by one ballot
    // per row against a warp-uniform running count (skewed passes), 5 the
    // early count's atomics return the in-warp ranks (lane-ordered, packed
    // 16-bit counters) and ranking is one lookup of the warp's digit base --
    // for full TMA-landed tiles; other tiles rank as 1. 6 is 5 with 2's hot
    // digit (ranked by ballots in the early phase), other tiles rank as 2.
    constexpr bool ER = (RANK == 5 || RANK == 6) && FULL && FROM_SMEM;
    constexpr int RB = RANK == 5 ? 1 : (RANK == 6 ? 2 : RANK);  // non-ER behaviour
    // ELB (experiment, off): the look-back runs right after the digit section
    // (its warps rank afterwards), so inclusive prefixes are published
    // earlier. Measured per 2^28-key u32 pass: 0.726 ms off, 0.86 on, 0.81 on
    // with separate staging -- the ranking hides the look-back's latency
    constexpr bool ELB = ER && B2S_EARLY_LB;
    (void)prof_acc;
    (void)prof_t;
    (void)hot;
    using W = LookbackWord<LB>;
    using OFF = typename TileShared<LB>::OFF;
    constexpr int WARPS = THREADS / 32;
    constexpr int WSEG = 32 * ITEMS;
    constexpr int LOOKBACK = B2S_LB_STEP;  // predecessors read per synchronous look-back step
    constexpr int PRE = W::kPrefetch;      // predecessors prefetched before ranking
    constexpr int HALF = kRadix / 2;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const uint32_t cnt_a = smem_addr(s_cnt + warp * HALF);
    // staging (scatter) target: the landing buffer itself, or with SEP the
    // other tile buffer (then the landing buffer is only ever read here)
    const uint32_t keys_a = smem_addr(sbuf);
    const uint32_t vals_a = smem_addr(svbuf);
    const uint32_t match_a = smem_addr(s_match + warp * kRadix);
    (void)match_a;
    const uint32_t dummy_a = smem_addr(sh.dummy + lane);

    // ---- load: warp w owns keys [w*WSEG, (w+1)*WSEG) of the tile; item j of
    // lane l is key j*32+l (coalesced / conflict-free; in-warp order == input order)
    U keys[ITEMS];
    uint32_t vals[VALS ? ITEMS : 1];
    uint32_t rr[ER ? (ITEMS + 1) / 2 : 1];  // RANK 5: packed in-warp ranks
    const uint32_t wbase = warp * WSEG;
    if constexpr (FROM_SMEM) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) keys[j] = kbuf[wbase + j * 32 + lane];
        if constexpr (VALS) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) vals[j] = vbuf[wbase + j * 32 + lane];
        }
    } else {
        const U* wsrc = src + tile_base + wbase + lane;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            if (FULL) keys[j] = __ldcs(wsrc + j * 32);
            else keys[j] = (wbase + j * 32 + lane < tile_valid) ? wsrc[j * 32] : U(0);
        }
        if constexpr (VALS) {
            const uint32_t* wv = vsrc + tile_base + wbase + lane;
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                if (FULL) vals[j] = __ldcs(wv + j * 32);
                else vals[j] = (wbase + j * 32 + lane < tile_valid) ? wv[j * 32] : 0u;
            }
        }
    }

    // ---- early counts: per-warp digit histogram. Even and odd digits count
    // into separate words with +1 increments (ATOMS.POPC.INC aggregates lanes
    // that hit the same counter); the digit section packs them into 16-bit
    // pairs for ranking.
    // RANK 5/6 (B2S_ECNT_IN_CNT): the packed early counts live in the warp's
    // own s_cnt segment (the digit section turns them into its lookup table in
    // place), so no other warp's data shares their words
    constexpr bool ECNT = ER && B2S_ECNT_IN_CNT;
    uint32_t* ecnt = ECNT ? s_cnt + warp * HALF : s_early + warp * kRadix;
    if constexpr (ER) {
        early_ranks<U, ITEMS, RANK == 6>(keys, rr, ecnt, shift, dxor, hot);
    } else {
        // each warp clears its own counters: 1 KB of the idle tile buffer
        // (nothing streams into it before this tile's look-back is done)
        uint4* z = reinterpret_cast<uint4*>(ecnt);
#pragma unroll
        for (int i = lane; i < kRadix / 4; i += 32) z[i] = make_uint4(0, 0, 0, 0);
        __syncwarp();
    }
    if constexpr (ER) {
        // ranked above
    } else if constexpr (RB == 2) {
        uint32_t hot_n = 0;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t d = digit_of(keys[j], shift, dxor);
            const bool valid = FULL || wbase + j * 32 + lane < tile_valid;
            const bool is_hot = valid && d == hot;
            hot_n += __popc(__ballot_sync(0xffffffffu, is_hot));
            if (valid && !is_hot) atomicAdd(ecnt + ((d & 1) * HALF + (d >> 1)), 1u);
        }
        if (lane == 0 && hot_n) atomicAdd(ecnt + ((hot & 1) * HALF + (hot >> 1)), hot_n);
    } else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t d = digit_of(keys[j], shift, dxor);
            if (FULL || wbase + j * 32 + lane < tile_valid) atomicAdd(ecnt + ((d & 1) * HALF + (d >> 1)), 1u);
        }
    }
    between();  // publish the next tile id
    __syncthreads();  // also: every warp has read its keys out of kbuf
    B2S_PHASE(1);
    // With the early counts in s_cnt the other tile buffer holds nothing but
    // the previous tile's staged keys, all written out once every warp has
    // passed the barrier above: the next tile streams in from here on (else
    // after the look-back). Separate staging buffers: after the key re-read.
    constexpr bool EARLY_CLAIM = ECNT && B2S_EARLY_CLAIM;
    if constexpr (EARLY_CLAIM && !SEP) claim_next();

    // ---- per digit pair (thread t < 128 owns digits 2t, 2t+1): exclusive
    // prefix over warps, tile counts, publish them at once
    uint32_t pair = 0;  // packed tile counts of the two digits
    if (tid < HALF) {
#pragma unroll 4
        for (int w = 0; w < WARPS; ++w) {
            uint32_t* e = s_early + w * kRadix;
            uint32_t c;
            if constexpr (ECNT) {
                c = s_cnt[w * HALF + tid];  // packed pair, replaced by the prefix below
            } else if constexpr (ER) {
                c = e[tid];  // packed pair; the region is cleared at the next tile's start
            } else {
                c = e[tid] | (e[HALF + tid] << 16);
                e[tid] = 0;
                e[HALF + tid] = 0;
            }
            s_cnt[w * HALF + tid] = pair;
            pair += c;
        }
        const uint32_t c0 = pair & 0xFFFFu, c1 = pair >> 16;
        if (ticket == nullptr) {
            LB* slot = lb_cur + (size_t)tile * kRadix + 2 * tid;
            const LB flag = tile == 0 ? W::kInc : W::kAgg;
            if constexpr (sizeof(LB) == 4 && B2S_LB_PAIR) {
                st_relaxed(reinterpret_cast<unsigned long long*>(slot),
                           (unsigned long long)(flag | (LB)c0) | ((unsigned long long)(flag | (LB)c1) << 32));
            } else {
                st_relaxed(slot, flag | (LB)c0);
                st_relaxed(slot + 1, flag | (LB)c1);
            }
        }
        uint32_t incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) sh.wsum[warp] = incl;
        sh.start[2 * tid] = incl - c0 - c1;  // partial (within warp)
        sh.start[2 * tid + 1] = incl - c1;
    }
    // start the look-back's first reads now (cp.async into shared memory, no
    // registers held) so their latency hides behind the ranking below. A stale
    // copy is harmless: a slot only moves 0 -> aggregate -> inclusive and every
    // non-zero state is valid; zeros are re-polled.
    if (tid < kRadix && tile > 0 && ticket == nullptr) {
#pragma unroll
        for (int i = 0; i < PRE; ++i) {
            if ((int64_t)tile - 1 - i >= 0)
                cp_async_lb(smem_addr(sh.lbw + i * kRadix + tid),
                            lb_cur + (size_t)(tile - 1 - i) * kRadix + tid);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // RANK 5/6: only the four scanning warps wait for each other here (named
    // barrier); the others go on to re-read their keys, and one full barrier
    // after the re-read covers both the finished digit section and the
    // in-place staging
    constexpr bool NAMED = ER && B2S_ERANK_RELOAD && B2S_NAMED_SCAN;
    if constexpr (NAMED) {
        if (tid < HALF) asm volatile("bar.sync 1, %0;" ::"n"(HALF) : "memory");
    } else {
        __syncthreads();
    }
    if (tid < HALF) {
        uint32_t base = 0;
#pragma unroll
        for (int w = 0; w < HALF / 32; ++w) base += (w < warp) ? sh.wsum[w] : 0u;
        const uint32_t s0 = sh.start[2 * tid] + base, s1 = sh.start[2 * tid + 1] + base;
        sh.start[2 * tid] = s0;
        sh.start[2 * tid + 1] = s1;
        const uint32_t add = s0 | (s1 << 16);
#pragma unroll 4
        for (int w = 0; w < WARPS; ++w) s_cnt[w * HALF + tid] += add;
    }
    if constexpr (!NAMED) __syncthreads();
    // ---- decoupled look-back: one lane per digit. The first PRE predecessors
    // were fetched before ranking; later steps read LOOKBACK at a time
    // (independent loads) in a warp-uniform loop. Each lane publishes its
    // inclusive prefix the moment it is known.
    auto lookback = [&]() {
        if constexpr (sizeof(LB) == 4 && B2S_LB_PAIR) {
            if (ticket == nullptr) {
                const int lt = tid - 32 * B2S_LB_WARP0;  // pair index of this thread
                if (lt >= 0 && lt < kRadix / 2) {
                    const uint32_t d0 = 2 * lt, d1 = 2 * lt + 1;
                    const uint32_t s0 = sh.start[d0], s1 = sh.start[d1];
                    const uint32_t s2 = d1 + 1 < kRadix ? sh.start[d1 + 1] : (uint32_t)tile_valid;
                    const unsigned long long rest = sh.n - tile_base;
                    const uint32_t h0 = sh.dcount[d0], h1 = sh.dcount[d1];
                    unsigned long long e0, e1;
                    lookback_exclusive_pair(tile, reinterpret_cast<uint32_t*>(lb_cur), s1 - s0, s2 - s1,
                                            h0 > rest ? h0 - rest : 0, h1 > rest ? h1 - rest : 0,
                                            B2S_LB_SKIP_EMPTY && h0 == 0 && h1 == 0, e0, e1);
                    gbase_out[d0] = (OFF)(sh.goff[d0] + e0 - s0);
                    gbase_out[d1] = (OFF)(sh.goff[d1] + e1 - s1);
                }
                return;
            }
        }
        if (tid < kRadix) {
            const uint32_t mycount = (tid + 1 < kRadix ? sh.start[tid + 1] : (uint32_t)tile_valid) - sh.start[tid];
            // 32-bit words: digit tid's keys in tiles >= tile number at most
            // the keys from tile_base on, so its exclusive prefix is at
            // least dcount - (n - tile_base); the prefix is at most
            // min(tile_base, dcount), a window narrower than 2^30 (below)
            unsigned long long lo = 0;
            bool empty_digit = false;
            if constexpr (sizeof(LB) == 4) {
                const unsigned long long rest = sh.n - tile_base;
                lo = sh.dcount[tid] > rest ? sh.dcount[tid] - rest : 0;
                empty_digit = B2S_LB_SKIP_EMPTY && sh.dcount[tid] == 0;
            }
            // keys-only first pass: no order to keep among equal digits, so
            // a tile's offsets come from one fetch-and-add per digit in
            // arrival order -- no look-back chain
            const unsigned long long excl = ticket != nullptr ? atomicAdd(ticket + tid, (unsigned long long)mycount)
                                                              : lookback_exclusive<LB>(tile, lb_cur, sh.lbw, mycount, lo, empty_digit);
            gbase_out[tid] = (OFF)(sh.goff[tid] + excl - sh.start[tid]);
        }
    };
#if B2S_ERANK_RELOAD
    if constexpr (ER) {
        // only the packed ranks were held across the digit section; the keys
        // come back from the landing buffer, and the in-place scatter starts
        // once every warp holds them
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) keys[j] = kbuf[wbase + j * 32 + lane];
        if constexpr (VALS) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) vals[j] = vbuf[wbase + j * 32 + lane];
        }
        // in-place staging: all reads first (and with NAMED the digit section's end)
        if constexpr (!SEP || NAMED) __syncthreads();
        if constexpr (EARLY_CLAIM && SEP) claim_next();
    }
#endif
    if constexpr (ELB) lookback();
    B2S_PHASE(2);

    // ---- rank within the tile and stage digit-sorted in shared memory. The
    // warp's counters start at its offset for each digit; item j of lane l
    // precedes item j of lane l+1 and item j+1 of any lane (input order), so
    // ranks are stable. The highest lane of each digit group claims the group's
    // slots with one atomic and shuffles the base to its peers.
    const uint32_t lanemask_lt = (1u << lane) - 1u;
    if constexpr (ER) {
        // slot = tile start of the digit + this warp's prefix (s_cnt, packed)
        // + the in-warp rank
        const uint32_t* wc = s_cnt + warp * HALF;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
#if B2S_ERANK_RELOAD
            const uint32_t d = digit_of(keys[j], shift, dxor);
#else
            // recomputed behind an opaque op: keeping the early phase's digits
            // live across the digit section would cost ITEMS more registers
            uint32_t w, d;
            if constexpr (sizeof(U) == 4) w = (uint32_t)keys[j];
            else w = shift >= 32 ? (uint32_t)((unsigned long long)keys[j] >> 32) : (uint32_t)keys[j];
            asm volatile("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(w), "r"(0x4440u | ((shift >> 3) & 3)));
            d ^= dxor;
#endif
            const uint32_t r = ((wc[d >> 1] >> (16 * (d & 1))) & 0xFFFFu) + ((rr[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
            sts_key(keys_a + swz<sizeof(U), SWZ>(r) * (uint32_t)sizeof(U), keys[j]);
            if constexpr (VALS) sts_key(vals_a + 4 * swz<4, SWZ>(r), vals[j]);
        }
    } else if constexpr (RB == 2 && FULL) {
        // hot lanes: the warp's running offset of the hot digit (nobody
        // else touches its counter) plus the lanes below in this row
        uint32_t hot_run = (s_cnt[warp * HALF + (hot >> 1)] >> (16 * (hot & 1))) & 0xFFFFu;
        constexpr int B = 4;
#pragma unroll
        for (int j0 = 0; j0 < ITEMS; j0 += B) {
            uint32_t old[B], s16[B], r[B];
            bool h[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (j0 + b < ITEMS) {
                    const uint32_t d = digit_of(keys[j0 + b], shift, dxor);
                    h[b] = d == hot;
                    const uint32_t hm = __ballot_sync(0xffffffffu, h[b]);
                    r[b] = hot_run + __popc(hm & lanemask_lt);
                    hot_run += __popc(hm);
                    s16[b] = 16 * (d & 1);
                    old[b] = atom_add_shared_if(!h[b], cnt_a + 4 * (d >> 1), 1u << s16[b]);
                }
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (j0 + b < ITEMS) {
                    const uint32_t rr = h[b] ? r[b] : (old[b] >> s16[b]) & 0xFFFFu;
                    sts_key(keys_a + swz<sizeof(U), SWZ>(rr) * (uint32_t)sizeof(U), keys[j0 + b]);
                    if constexpr (VALS) sts_key(vals_a + 4 * swz<4, SWZ>(rr), vals[j0 + b]);
                }
            }
        }
    } else if constexpr (RB == 1 && FULL) {
        // atomic ranking in batches of 4 items: the batch's atomics are
        // independent (the warp's shared accesses stay in program order, so
        // the counters advance exactly as item by item) and their latencies
        // overlap before the scatters consume them
        constexpr int B = 4;
#pragma unroll
        for (int j0 = 0; j0 < ITEMS; j0 += B) {
            uint32_t old[B], s16[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (j0 + b < ITEMS) {
                    const uint32_t d = digit_of(keys[j0 + b], shift, dxor);
                    s16[b] = 16 * (d & 1);
                    old[b] = atom_add_shared(cnt_a + 4 * (d >> 1), 1u << s16[b]);
                }
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (j0 + b < ITEMS) {
                    const uint32_t r = (old[b] >> s16[b]) & 0xFFFFu;
                    sts_key(keys_a + swz<sizeof(U), SWZ>(r) * (uint32_t)sizeof(U), keys[j0 + b]);
                    if constexpr (VALS) sts_key(vals_a + 4 * swz<4, SWZ>(r), vals[j0 + b]);
                }
            }
        }
    } else
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const bool valid = FULL || (wbase + j * 32 + lane < tile_valid);
        const uint32_t d = valid ? digit_of(keys[j], shift, dxor) : (uint32_t)kRadix;
        uint32_t r;
        if constexpr (RB >= 1) {
            // lane-ordered shared atomics: lanes adding to the same counter in one
            // warp instruction receive old values in ascending lane order on this
            // device (verified at context creation by b2s::probe_lane_order), so
            // the returned count is directly the stable rank -- no match needed
            const uint32_t sh16 = 16 * (d & 1);
            const uint32_t a = cnt_a + 4 * ((d >> 1) & (HALF - 1));
            const uint32_t old = FULL ? atom_add_shared(a, 1u << sh16)
                                      : atom_add_shared(valid ? a : dummy_a, valid ? 1u << sh16 : 0u);
            r = (old >> sh16) & 0xFFFFu;
        } else {
        uint32_t peers;
        if (MATCH_SMEM && (B2S_MATCH_HYBRID == 1 || (j % B2S_MATCH_HYBRID) != 0)) {
            // odd items: OR-mask match through shared memory (LSU pipe) to
            // balance the ALU pipe the ballot match saturates
            peers = match_smem(valid, match_a + 4 * (d & (kRadix - 1)), 1u << lane);
        } else {
            peers = match_digit<FULL ? 8 : 9>(d);
        }
        const uint32_t below = __popc(peers & lanemask_lt);
        const int leader = 31 - __clz(peers);
        const uint32_t sh16 = 16 * (d & 1);
        // every lane issues the atomic (no divergent branch: a branch costs two
        // ADU-pipe reconvergence ops per item); non-leaders add 0 to a private
        // dummy word so they neither conflict with nor change the counters
        const bool claim = valid && lane == leader;
        const uint32_t old = atom_add_shared(claim ? cnt_a + 4 * ((d >> 1) & (HALF - 1)) : dummy_a,
                                             claim ? (below + 1) << sh16 : 0u);
        const uint32_t base = (__shfl_sync(0xffffffffu, old, leader) >> sh16) & 0xFFFFu;
        r = base + below;
        }
        if (valid) {
            sts_key(keys_a + swz<sizeof(U), SWZ>(r) * (uint32_t)sizeof(U), keys[j]);
            if constexpr (VALS) sts_key(vals_a + 4 * swz<4, SWZ>(r), vals[j]);
        }
    }
    B2S_PHASE(3);

    if constexpr (!ELB) lookback();
    __syncthreads();
    B2S_PHASE(4);
    if constexpr (!EARLY_CLAIM) claim_next();

    // ---- write runs of equal digits; clear this warp's counters (RANK 5
    // overwrites them in the digit section)
    if constexpr (!ER) {
#pragma unroll
        for (int i = lane; i < HALF; i += 32) s_cnt[warp * HALF + i] = 0;
    }
    writeout_tile<U, VALS, LB, THREADS, ITEMS, RB == 2, SWZ>(sbuf, svbuf, gbase_out, tile_valid, dst,
                                                               vdst, shift, dxor, nd);
}

template <typename U, bool VALS, typename LB, int THREADS, int ITEMS, int MINB, int RANK>
__global__ void __launch_bounds__(THREADS, MINB) onesweep_kernel(RadixPlan* __restrict__ plan,
                                                                 RadixCounters* __restrict__ ctr,
                                                                 int slot, uint64_t n,
                                                                 uint32_t ntiles,
                                                                 LB* __restrict__ lb_cur,
                                                                 LB* __restrict__ lb_next,
                                                                 uint64_t skew_limit) {
    using SM = OnesweepSmem<U, VALS, THREADS, ITEMS>;
    constexpr int TILE = SM::TILE;
    static_assert(THREADS >= kRadix, "one thread per digit is required");
    static_assert(TILE < 65536, "packed 16-bit warp counters");
    // Full tiles of RANK 1, 2 and 4 rank by the early count's returned in-warp
    // ranks plus one lookup (onesweep_tile RANK 5; B2S_ERANK=0 restores the
    // second atomic pass: 0.811 -> 0.774 ms per 2^28-key u32 pass).
    // RANK: 0 ballots, 1 atomics (one kernel per pass), or one of three
    // kernels launched back to back per pass, exactly one of which runs it:
    //   2  atomics, unless the pass is skewed or the input structured;
    //   3  skewed pass (a digit holds more than skew_limit keys): same-address
    //      shared atomics serialise across the lanes that share a digit, so
    //      that digit is counted and ranked by ballots, the rest by atomics;
    //   4  structured input, pass not skewed: atomics + swizzled staging.
    // 3 and 4 are programmatic dependents of their predecessor: their CTAs
    // take the SMs as the predecessor's drain, and the ones not suited to the
    // pass exit at once. What they decide on (the pass's histogram, the
    // prologue's order statistic) was final before 2 started.
    constexpr int TR = RANK == 3 ? (B2S_ERANK ? 6 : 2) : (RANK >= 1 ? (B2S_ERANK ? 5 : 1) : 0);
    // separate landing / staging buffers: measured per 2^28-key u32 pass,
    // uniform keys 0.776 ms in place vs 0.794 separate, ascending (the
    // structured twin) 0.709 vs 0.699 -- so only the structured twin uses it
    constexpr bool SEP = TR == 5 && (RANK == 4 || B2S_SEP > 1) && B2S_SEP;
    constexpr bool SWZ = RANK == 4;
    if constexpr (RANK == 2 || RANK == 3)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    const int na = plan->num_active;
    if (slot >= na) return;
    const int tid = threadIdx.x;
    unsigned long long c = 0;  // this thread's digit count of the pass
    if (tid < kRadix) c = plan->hist[slot][tid];
    uint32_t hot = 0;  // the pass's most frequent digit (RANK 3)
    if constexpr (RANK >= 2) {
        const bool skewed = __syncthreads_or(tid < kRadix && c > skew_limit) != 0;
        const bool structured = plan->structured != 0;
        const int mode = skewed ? 3 : (structured ? 4 : 2);
        if (mode != RANK) return;
        if constexpr (RANK >= 3) asm volatile("griddepcontrol.wait;" ::: "memory");
        if constexpr (RANK == 3) {
            __shared__ unsigned long long s_hot;
            if (tid == 0) s_hot = 0;
            __syncthreads();
            if (tid < kRadix) atomicMax(&s_hot, (c << 8) | (unsigned long long)tid);
            __syncthreads();
            hot = (uint32_t)(s_hot & 0xFF);
        }
    }

    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem);
    // Tile buffer selection. Selected arithmetically (twins), every access
    // through them is a shared-memory LDS/STS; through an indexed pointer
    // array (regular kernel) the pointers live in local memory and the tile
    // loads and write-out reads are generic LD.E. Measured per 2^28-key u32
    // sort: regular kernel 3.455 ms with the array vs 3.535 ms arithmetic
    // (register allocation), twins faster arithmetic (sorted 2^27: 1.75 ->
    // 1.63 ms, Zipf 1.52 -> 1.48 ms).
    constexpr bool ARITH = RANK >= B2S_ARITH_MIN_RANK;
    struct Bufs {
        unsigned char* base;
        U* arr[2];
        __device__ __forceinline__ U* operator[](int b) const {
            if constexpr (ARITH) return reinterpret_cast<U*>(base + SM::kCnt + (b ? SM::kKeys : 0));
            else return arr[b];
        }
    };
    struct VBufs {
        unsigned char* base;
        uint32_t* arr[2];
        __device__ __forceinline__ uint32_t* operator[](int b) const {
            if constexpr (ARITH)
                return reinterpret_cast<uint32_t*>(base + SM::kCnt + 2 * SM::kKeys + (b ? SM::kVals : 0));
            else return arr[b];
        }
    };
    const Bufs kbuf{smem, {reinterpret_cast<U*>(smem + SM::kCnt),
                           reinterpret_cast<U*>(smem + SM::kCnt + SM::kKeys)}};
    const VBufs vbuf{smem, {reinterpret_cast<uint32_t*>(smem + SM::kCnt + 2 * SM::kKeys),
                            reinterpret_cast<uint32_t*>(smem + SM::kCnt + 2 * SM::kKeys + SM::kVals)}};
    __shared__ TileShared<LB> sh;
    __shared__ typename TileShared<LB>::OFF s_gbase[kRadix];

    const int shift = 8 * plan->digit[slot];
    const uint32_t dxor = plan->dxor[slot];
    // a keys-only sort's first pass need not be stable: equal keys are
    // indistinguishable and no earlier pass's order is to be kept
    unsigned long long* const ticket = (!VALS && slot == 0 && B2S_TICKET_FIRST) ? ctr->ticket : nullptr;
    const bool zero_next = slot + 1 < na;  // the last pass has no successor to zero words for
    const U* src = static_cast<const U*>(plan->ksrc[slot]);
    U* dst = static_cast<U*>(plan->kdst[slot]);
    const uint32_t* vsrc = plan->vsrc[slot];
    uint32_t* vdst = plan->vdst[slot];
    NextDigit nd;
    nd.on = slot + 1 < na && !plan->all_hist;
    nd.shift = nd.on ? 8 * plan->digit[slot + 1] : 0;
    nd.dxor = nd.on ? plan->dxor[slot + 1] : 0u;
    nd.hist = sh.nhist;
    // TMA needs 16-byte aligned global sources (tiles are 16-byte multiples)
    const bool tma = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                     (!VALS || (reinterpret_cast<uintptr_t>(vsrc) & 15) == 0);
    const uint32_t mbar_a[2] = {smem_addr(&sh.mbar[0]), smem_addr(&sh.mbar[1])};
    const uint32_t tx_bytes = (uint32_t)(SM::kKeys + SM::kVals);

    auto prefetch = [&](uint32_t t, int b) {  // one thread only
        if (tma && t < ntiles && n - (uint64_t)t * TILE >= (uint64_t)TILE) {
            fence_proxy_async();
            mbar_expect_tx(mbar_a[b], tx_bytes);
            bulk_g2s(smem_addr(kbuf[b]), src + (uint64_t)t * TILE, (uint32_t)SM::kKeys, mbar_a[b]);
            if constexpr (VALS)
                bulk_g2s(smem_addr(vbuf[b]), vsrc + (uint64_t)t * TILE, (uint32_t)SM::kVals, mbar_a[b]);
        }
    };

    // global digit offsets of this slot: exclusive scan of its histogram
    if (tid < kRadix) {
        unsigned long long incl = c;
        const int lane = tid & 31;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) sh.wsum64[tid >> 5] = incl;
        sh.goff[tid] = (typename TileShared<LB>::OFF)(incl - c);
        if constexpr (sizeof(LB) == 4) sh.dcount[tid] = (uint32_t)c;
        if (tid == 0) sh.n = n;
        sh.nhist[tid] = 0;
    }
    for (int i = tid; i < SM::WARPS * (kRadix / 2); i += THREADS) s_cnt[i] = 0;
    if (tid == THREADS - 1) {
        mbar_init(mbar_a[0], 1);
        mbar_init(mbar_a[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t t = atomicAdd(&plan->tile_counter[slot], 1u);
        sh.tile[0] = t;
        prefetch(t, 0);
    }
    __syncthreads();
    if (tid < kRadix) {
        unsigned long long base = 0;
#pragma unroll
        for (int w = 0; w < kRadix / 32; ++w) base += (w < (tid >> 5)) ? sh.wsum64[w] : 0ull;
        sh.goff[tid] += (typename TileShared<LB>::OFF)base;
    }

    int cur = 0;
    uint32_t parity = 0;  // bit b: phase parity of buffer b's mbarrier
    unsigned long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long prof_t = clock64();
    (void)prof_t;
    for (;;) {
        const uint32_t tile = sh.tile[cur];
        if (tile >= ntiles) break;
        // claim the next tile and stream it in during this tile's write-out
        // (by a thread that sits out the look-back); the id is fetched now
        // (its atomic's latency hides behind the early counts)
        uint32_t next_t = 0;
        if (tid == THREADS - 1) next_t = atomicAdd(&plan->tile_counter[slot], 1u);
        // SEP: tiles always land in buffer 0 and are staged in buffer 1
        // (which also holds the early counts); else the two alternate and
        // each tile is staged in place
        const int lb_ = SEP ? 0 : cur;
        const int sb_ = SEP ? 1 : cur;
        // the next tile id is published before the early-count barrier (so
        // every thread knows it at this tile's end), its copy is issued after
        // the look-back (the buffer is free then)
        auto publish = [&]() {
            if (tid == THREADS - 1) sh.tile[cur ^ 1] = next_t;
        };
        auto claim = [&]() {
            if (tid == THREADS - 1) prefetch(next_t, SEP ? 0 : cur ^ 1);
        };
        const uint64_t tile_base = (uint64_t)tile * TILE;
        const uint64_t rem = n - tile_base;
        if (zero_next && tid < kRadix) lb_next[(size_t)tile * kRadix + tid] = 0;  // the next slot's words
        uint32_t* idle = reinterpret_cast<uint32_t*>(kbuf[SEP ? 1 : cur ^ 1]);
        if (rem >= (uint64_t)TILE) {
            if (tma) {
                mbar_wait(mbar_a[lb_], (parity >> lb_) & 1u);
                parity ^= 1u << lb_;
                B2S_PHASE(0);
                onesweep_tile<U, VALS, LB, THREADS, ITEMS, true, true, TR, SWZ, SEP>(
                    claim, publish, s_gbase, tile, TILE, tile_base, src, dst, vsrc, vdst, lb_cur, ticket, shift,
                    dxor, nd, s_cnt, kbuf[lb_], vbuf[lb_], kbuf[sb_], vbuf[sb_], idle, idle, sh, prof_acc, prof_t,
                    hot);
            } else {
                onesweep_tile<U, VALS, LB, THREADS, ITEMS, true, false, TR, SWZ, SEP>(
                    claim, publish, s_gbase, tile, TILE, tile_base, src, dst, vsrc, vdst, lb_cur, ticket, shift,
                    dxor, nd, s_cnt, kbuf[lb_], vbuf[lb_], kbuf[sb_], vbuf[sb_], idle, idle, sh, prof_acc, prof_t,
                    hot);
            }
        } else {
            onesweep_tile<U, VALS, LB, THREADS, ITEMS, false, false, TR, SWZ, SEP>(
                claim, publish, s_gbase, tile, (uint32_t)rem, tile_base, src, dst, vsrc, vdst, lb_cur, ticket,
                shift, dxor,
                nd, s_cnt, kbuf[lb_], vbuf[lb_], kbuf[sb_], vbuf[sb_], idle, idle, sh, prof_acc, prof_t, hot);
        }
        // Between two full TMA tiles of the early-rank kernels no barrier is
        // needed: the next tile's early counts go to each warp's own s_cnt
        // segment and it lands in the other buffer, and its first barrier
        // (after the early counts) is only passed once every warp has
        // finished this write-out. Any other next tile (partial: early counts
        // in this staging buffer; none: the CTA's final reductions) waits.
        {
            bool skip = false;
            if constexpr ((TR == 5 || TR == 6) && B2S_ECNT_IN_CNT && B2S_ERANK_RELOAD) {
                const uint32_t nt = sh.tile[cur ^ 1];
                skip = tma && nt < ntiles && n - (uint64_t)nt * TILE >= (uint64_t)TILE;
            }
            if (!skip) __syncthreads();
        }
        B2S_PHASE(5);
        cur ^= 1;
    }
#ifdef B2S_PHASE_PROFILE
    if (tid == 0 || tid == THREADS - 1)
        for (int k = 0; k < 8; ++k) atomicAdd(&b2s_phase_cycles[tid == 0 ? 0 : 1][k], prof_acc[k]);
#endif
    // hand the next slot's digit counts to global memory once per CTA
    if (nd.on && tid < kRadix && sh.nhist[tid])
        atomicAdd(&ctr->hist[slot + 1][tid], (unsigned long long)sh.nhist[tid]);
}

// n elements of T, 16-byte vectors where source and destination share their
// 16-byte phase (the aligned middle), elements elsewhere
template <typename T>
__device__ __forceinline__ void copy_elems(const T* __restrict__ s, T* __restrict__ d, uint64_t n) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr uint32_t V = 16 / sizeof(T);
    const uint32_t ps = (uint32_t)((reinterpret_cast<uintptr_t>(s) & 15) / sizeof(T));
    const uint32_t pd = (uint32_t)((reinterpret_cast<uintptr_t>(d) & 15) / sizeof(T));
    if (ps != pd) {
        for (uint64_t i = tid; i < n; i += stride) d[i] = s[i];
        return;
    }
    const uint64_t head = std::min<uint64_t>((V - ps) % V, n);
    const uint64_t nv = (n - head) / V;
    const uint4* __restrict__ sv = reinterpret_cast<const uint4*>(s + head);
    uint4* __restrict__ dv = reinterpret_cast<uint4*>(d + head);
    for (uint64_t i = tid; i < nv; i += stride) __stcs(dv + i, __ldcs(sv + i));
    for (uint64_t i = tid; i < head; i += stride) d[i] = s[i];
    for (uint64_t i = head + nv * V + tid; i < n; i += stride) d[i] = s[i];
}

template <typename T>
__device__ __forceinline__ uint4 reverse_vec(uint4 q) {
    if constexpr (sizeof(T) == 4) return make_uint4(q.w, q.z, q.y, q.x);
    else return make_uint4(q.z, q.w, q.x, q.y);
}

// d[i] = s[n-1-i]; s == d reverses in place. 16-byte vectors when n is a whole
// number of them and both arrays are aligned, elements otherwise.
template <typename T>
__device__ __forceinline__ void reverse_elems(const T* s, T* d, uint64_t n) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr uint32_t V = 16 / sizeof(T);
    const bool vec = n % V == 0 && ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0;
    if (s != d) {
        if (vec) {
            const uint64_t nv = n / V;
            const uint4* sv = reinterpret_cast<const uint4*>(s);
            uint4* dv = reinterpret_cast<uint4*>(d);
            for (uint64_t i = tid; i < nv; i += stride) __stcs(dv + (nv - 1 - i), reverse_vec<T>(__ldcs(sv + i)));
        } else {
            for (uint64_t i = tid; i < n; i += stride) d[n - 1 - i] = s[i];
        }
        return;
    }
    if (vec) {
        const uint64_t nv = n / V;
        uint4* dv = reinterpret_cast<uint4*>(d);
        for (uint64_t i = tid; i < (nv + 1) / 2; i += stride) {
            const uint64_t j = nv - 1 - i;
            const uint4 a = dv[i], b = dv[j];
            dv[j] = reverse_vec<T>(a);
            if (i != j) dv[i] = reverse_vec<T>(b);
        }
    } else {
        for (uint64_t i = tid; i < n / 2; i += stride) {
            const T a = d[i], b = d[n - 1 - i];
            d[i] = b;
            d[n - 1 - i] = a;
        }
    }
}

template <typename U>
__global__ void radix_copy_kernel(const RadixPlan* __restrict__ plan, uint64_t n, int with_vals) {
    if (!plan->do_copy) return;
    if (plan->do_copy == 2) {
        reverse_elems(static_cast<const U*>(plan->copy_ksrc), static_cast<U*>(plan->copy_kdst), n);
        if (with_vals) reverse_elems(plan->copy_vsrc, plan->copy_vdst, n);
        return;
    }
    copy_elems(static_cast<const U*>(plan->copy_ksrc), static_cast<U*>(plan->copy_kdst), n);
    if (with_vals) copy_elems(plan->copy_vsrc, plan->copy_vdst, n);
}

// Orders the ties of an upper-digits-first sort (see radix_plan_kernel): the
// array is sorted (stably) by the keys' upper halves; the thread at the first
// element of a run of equal upper halves walks the run and, when its lower
// halves are not already ascending, sorts it in place by insertion (stable;
// payloads move with their keys). Only the run's owner writes it, and what the
// other threads read of it -- upper halves -- does not change. Runs longer
// than kFixScan, or unsorted ones longer than kFixSort, raise plan->fix_flag.
constexpr uint32_t kFixScan = 4096, kFixSort = 32;

// One tie run starting at element i (see topfirst_fixup_kernel).
template <bool VALS>
__device__ __noinline__ void fixup_run(RadixPlan* plan, unsigned long long* keys, uint32_t* vals,
                                       uint64_t n, uint64_t i) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(keys);  // w[2i]: lower half, w[2i+1]: upper
    {
        // runs of two, nearly all of them: three independent loads, at most one swap
        const unsigned long long k0 = keys[i], k1 = keys[i + 1];
        const unsigned long long k2 = i + 2 < n ? keys[i + 2] : ~k0;
        if ((uint32_t)(k2 >> 32) != (uint32_t)(k0 >> 32)) {
            if ((uint32_t)k0 > (uint32_t)k1) {
                keys[i] = k1;
                keys[i + 1] = k0;
                if constexpr (VALS) {
                    const uint32_t v0 = vals[i], v1 = vals[i + 1];
                    vals[i] = v1;
                    vals[i + 1] = v0;
                }
            }
            return;
        }
    }
    const uint32_t hi = w[2 * i + 1];
    uint64_t j = i + 1;
    uint32_t prev = w[2 * i];
    bool sorted = true, ended = false;
    while (j < n && j - i < kFixScan) {
        if (w[2 * j + 1] != hi) {
            ended = true;
            break;
        }
        const uint32_t lo = w[2 * j];
        sorted = sorted && prev <= lo;
        prev = lo;
        ++j;
    }
    if (!ended && j < n && w[2 * j + 1] == hi) {  // longer than the scan window
        plan->fix_flag = 1;
        return;
    }
    if (sorted) return;
    const uint32_t len = (uint32_t)(j - i);
    if (len > kFixSort) {
        plan->fix_flag = 1;
        return;
    }
    for (uint32_t a = 1; a < len; ++a) {
        const unsigned long long x = keys[i + a];
        uint32_t vx = 0;
        if constexpr (VALS) vx = vals[i + a];
        uint32_t b = a;
        while (b > 0 && (uint32_t)keys[i + b - 1] > (uint32_t)x) {
            keys[i + b] = keys[i + b - 1];
            if constexpr (VALS) vals[i + b] = vals[i + b - 1];
            --b;
        }
        keys[i + b] = x;
        if constexpr (VALS) vals[i + b] = vx;
    }
}

// Each lane reads four consecutive keys (two 16-byte loads) per step and gets
// its neighbours' boundary upper halves by shuffle; the lanes that find a run
// start (upper half differs from the predecessor's and equals the
// successor's) handle their runs.
template <bool VALS>
__global__ void __launch_bounds__(256) topfirst_fixup_kernel(RadixPlan* __restrict__ plan,
                                                             unsigned long long* keys, uint32_t* vals,
                                                             uint64_t n) {
    if (!plan->topfirst) return;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(keys);
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    if ((reinterpret_cast<uintptr_t>(keys) & 15) != 0) {  // unaligned: one element per thread
        const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += stride) {
            const uint32_t hi = w[2 * i + 1];
            if (w[2 * i + 3] == hi && (i == 0 || w[2 * i - 1] != hi)) fixup_run<VALS>(plan, keys, vals, n, i);
        }
        return;
    }
    const uint4* kv = reinterpret_cast<const uint4*>(keys);
    for (uint64_t base = warp * 128; base < n; base += nwarps * 128) {  // warp-uniform trips
        const uint64_t i0 = base + 4 * (uint64_t)lane;
        uint32_t t[6];  // upper halves of elements i0-1 .. i0+4 (0/1 sentinels past the ends)
        uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
        if (i0 + 1 < n) a = kv[i0 / 2];
        else if (i0 < n) a.y = w[2 * i0 + 1];
        if (i0 + 3 < n) b = kv[i0 / 2 + 1];
        else if (i0 + 2 < n) b.y = w[2 * (i0 + 2) + 1];
        t[1] = a.y;
        t[2] = a.w;
        t[3] = b.y;
        t[4] = b.w;
        const uint32_t up = __shfl_up_sync(0xffffffffu, t[4], 1);
        const uint32_t dn = __shfl_down_sync(0xffffffffu, t[1], 1);
        t[0] = lane > 0 ? up : (i0 > 0 ? w[2 * i0 - 1] : ~t[1]);
        t[5] = lane < 31 ? dn : (i0 + 4 < n ? w[2 * (i0 + 4) + 1] : 0u);
        uint32_t starts = 0;  // bit e: element i0 + e opens a run
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint64_t i = i0 + e;
            if (i + 1 < n && t[e + 1] == t[e + 2] && (i == 0 || t[e] != t[e + 1])) starts |= 1u << e;
        }
        while (starts) {  // one call site: the lanes with a run handle theirs together
            const int e = __ffs(starts) - 1;
            starts &= starts - 1;
            fixup_run<VALS>(plan, keys, vals, n, i0 + e);
        }
    }
}

// B2S_TOPFIRST=0 turns the upper-digits-first path of 8-byte keys off
bool topfirst_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("B2S_TOPFIRST");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}
constexpr uint64_t kTopFirstMinKeys = 1ull << 22, kTopFirstMaxKeys = 1ull << 31;

// B2S_ALL_HIST: 1 (default) all-digit prologue for 4-byte keys, 2 also for
// 8-byte keys, 0 never (each next digit is counted inside the passes)
int all_hist_mode() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("B2S_ALL_HIST");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// A pass is skewed when one digit holds more than n >> B2S_SKEW_SHIFT keys
// (default 3: an eighth; 64 never). Measured per 2^27-key pass: uniform keys
// 0.42 ms regular / 0.52 ms hot-digit path; Zipf(1.2) keys, top digit ~20%:
// 0.557 / 0.525; top digit ~75%: 1.00-1.14 / 0.39-0.48.
constexpr uint64_t kTwinMinKeys = 1ull << 21;

uint64_t skew_limit(uint64_t n) {
    static int sh = -1;
    if (sh < 0) {
        const char* e = getenv("B2S_SKEW_SHIFT");
        sh = e ? atoi(e) : 3;
    }
    return sh >= 64 ? ~0ull : (n >> sh);
}

template <typename U, bool VALS, typename LB, int THREADS, int ITEMS, int MINB, int RANK>
b2s_status launch_passes_cfg_r(b2s_ctx* ctx, RadixPlan* plan, RadixCounters* ctr, uint64_t n,
                               void* lb) {
    using SM = OnesweepSmem<U, VALS, THREADS, ITEMS>;
    constexpr int TILE = SM::TILE;
    constexpr size_t SMEM = SM::bytes;
    // the regular kernel and, for RANK 2, its skewed-pass and structured-input
    // twins (same tile and shared memory, so the same look-back layout)
    using Kern = void (*)(RadixPlan*, RadixCounters*, int, uint64_t, uint32_t, LB*, LB*, uint64_t);
    constexpr int NK = RANK == 2 ? 3 : 1;
    const Kern kern[3] = {onesweep_kernel<U, VALS, LB, THREADS, ITEMS, MINB, RANK>,
                          onesweep_kernel<U, VALS, LB, THREADS, ITEMS, MINB, 3>,
                          onesweep_kernel<U, VALS, LB, THREADS, ITEMS, MINB, 4>};
    static int occ[3] = {-1, -1, -1};  // per instantiation (one device type)
    static DeviceOnce once;
    B2S_TRY(once_per_device(once, ctx->device, [&]() -> b2s_status {
        for (int k = 0; k < NK; ++k) {
            B2S_CUDA(cudaFuncSetAttribute(kern[k], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)SMEM));
            int o = 0;
            B2S_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern[k], THREADS, SMEM));
            occ[k] = o > 0 ? o : 1;
            if (getenv("B2S_DEBUG")) {
                cudaFuncAttributes fa;
                cudaFuncGetAttributes(&fa, kern[k]);
                fprintf(stderr, "[b2s] onesweep<%zuB keys, vals=%d, %d thr, %d items, rank=%d>: dyn smem %zu + static %zu B, regs %d, %d CTA/SM\n",
                        sizeof(U), (int)VALS, THREADS, ITEMS, k == 0 ? RANK : k + 2, (size_t)SMEM,
                        (size_t)fa.sharedSizeBytes, fa.numRegs, occ[k]);
            }
        }
        return B2S_OK;
    }));
    const uint64_t ntiles64 = (n + TILE - 1) / TILE;
    const uint32_t ntiles = (uint32_t)ntiles64;
    LB* region[2] = {static_cast<LB*>(lb), static_cast<LB*>(lb) + (size_t)ntiles * kRadix};
    const int slots = (int)sizeof(U);
    const uint64_t skew = skew_limit(n);
    for (int s = 0; s < slots; ++s) {
        ctx->ev_pass[s] = record(ctx);
        for (int k = 0; k < NK; ++k) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((uint32_t)std::min<uint64_t>(ntiles64, (uint64_t)occ[k] * ctx->num_sms));
            lc.blockDim = dim3(THREADS);
            lc.dynamicSmemBytes = SMEM;
            lc.stream = ctx->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            lc.attrs = at;
            lc.numAttrs = k > 0 ? 1 : 0;  // the twins are programmatic dependents
            B2S_CUDA(cudaLaunchKernelEx(&lc, kern[k], plan, ctr, s, n, ntiles, region[s & 1],
                                        region[(s + 1) & 1], skew));
            note_launch();
        }
    }
    ctx->ev_pass[slots] = record(ctx);
    return B2S_OK;
}

template <typename U, bool VALS, typename LB, int THREADS, int ITEMS, int MINB>
b2s_status launch_passes_cfg(b2s_ctx* ctx, RadixPlan* plan, RadixCounters* ctr, uint64_t n,
                             void* lb) {
    // small sorts are bound by the chain of dependent launches, not by the
    // ranking: one kernel per pass (no skewed / structured twins)
    if (ctx->atomic_rank && n < kTwinMinKeys)
        return launch_passes_cfg_r<U, VALS, LB, THREADS, ITEMS, MINB, 1>(ctx, plan, ctr, n, lb);
    if (ctx->atomic_rank)
        return launch_passes_cfg_r<U, VALS, LB, THREADS, ITEMS, MINB, 2>(ctx, plan, ctr, n, lb);
    return launch_passes_cfg_r<U, VALS, LB, THREADS, ITEMS, MINB, 0>(ctx, plan, ctr, n, lb);
}

// Tile configuration of a sort: threads x items per CTA, CTAs per SM
// (registers must stay <= 65536 / (threads * minb) for minb CTAs per SM). The
// defaults fill the 2-CTA/SM shared-memory budget (two tile buffers of keys
// and payloads + 8 KB of counters per CTA). Alternatives measured in round 1
// (256x16x4, 1024x16x1, 512x20/22x2, 1024x24x1, 384x20x3, 256x24x4 for u32;
// 512x10 and 1024x12 for u32+payload and u64; 512x6/8 for u64+payload, and
// the software-pipelined and warp-specialised kernels) were all slower; their
// numbers are in DESIGN.md and their code in the history (commit d25c4e5).
struct TileCfg {
    int threads, items, minb;
};


TileCfg tile_cfg(int kbytes, bool vals, uint64_t n) {
    if (kbytes == 4 && vals) return {512, 12, 2};
    // small sorts (the partitions of cfg1) are latency-bound: smaller tiles,
    // more CTAs (2^20 keys, p = 4: 0.088 vs 0.095 ms per partitioned sort)
    if (kbytes == 4) return n < kTwinMinKeys ? TileCfg{512, 16, 2} : TileCfg{B2S_U32_THREADS, B2S_U32_ITEMS, B2S_U32_MINB};
    // 8-byte keys + payload: one 1024-thread CTA per SM with 8192-pair tiles
    // (per 2^28-pair pass 1.92 ms vs 1.97 for two 512-thread CTAs with
    // 4096-pair tiles)
    if (vals) return {1024, 8, 1};
    return {512, 12, 2};
}

template <typename U, bool VALS, typename LB>
b2s_status launch_passes(b2s_ctx* ctx, RadixPlan* plan, RadixCounters* ctr, uint64_t n, void* lb) {
    const TileCfg c = tile_cfg((int)sizeof(U), VALS, n);
    if constexpr (sizeof(U) == 4 && VALS) {
        return launch_passes_cfg<U, VALS, LB, 512, 12, 2>(ctx, plan, ctr, n, lb);
    } else if constexpr (sizeof(U) == 4) {
        if (c.items == 16) return launch_passes_cfg<U, VALS, LB, 512, 16, 2>(ctx, plan, ctr, n, lb);
        return launch_passes_cfg<U, VALS, LB, B2S_U32_THREADS, B2S_U32_ITEMS, B2S_U32_MINB>(ctx, plan, ctr, n, lb);
    } else if constexpr (VALS) {
        return launch_passes_cfg<U, VALS, LB, 1024, 8, 1>(ctx, plan, ctr, n, lb);
    } else {
        return launch_passes_cfg<U, VALS, LB, 512, 12, 2>(ctx, plan, ctr, n, lb);
    }
}

uint64_t lookback_tile(uint64_t n, int kbytes, bool vals) {
    const TileCfg c = tile_cfg(kbytes, vals, n);
    return (uint64_t)c.threads * c.items;
}

// 32-bit look-back words (2 flag bits, prefixes modulo 2^30) are exact when
// the window a tile's exclusive prefix can lie in is narrower than 2^30. For
// tile k of T keys and a digit of H keys the prefix E satisfies
//   max(0, H - (n - kT)) <= E <= min(kT, H),
// a window of at most min(kT, n - kT) <= n / 2 keys, equal to n / 2 only when
// kT = n / 2. So n <= 2^31 suffices, except n = 2^31 with T dividing 2^30.
// (64-bit words cost cfg3 -- 2^31 i32 -- 3.6% per pass.)
bool narrow_lookback_words(uint64_t n, uint64_t tile) {
    const uint64_t half = 1ull << 30;
    return n < 2 * half || (n == 2 * half && half % tile != 0);
}

template <typename U, bool VALS>
b2s_status radix_sort_t(b2s_ctx* ctx, bool is_signed, const void* kin, void* kout,
                        const uint32_t* vin, uint32_t* vout, uint64_t n, const SortScratch* sc,
                        int top_mode = 0) {
    // top_mode (own scratch only): 0 the plain sort; 1 the upper digits first
    // when the plan kernel finds the keys fit (plan[0]); 2 the full sort that
    // runs only if the fix-up raised plan[0].fix_flag (plan[1])
    constexpr int NP = sizeof(U);
    const uint32_t top_xor = is_signed ? 0x80u : 0u;
    const size_t lb_region = lookback_region_bytes(n, (int)sizeof(U), VALS);
    SortScratch own;
    if (sc == nullptr) {
        B2S_TRY(ctx->hist.ensure(sizeof(RadixCounters)));
        B2S_TRY(ctx->alt_keys.ensure(n * sizeof(U)));
        if (VALS) B2S_TRY(ctx->alt_vals.ensure(n * 4));
        B2S_TRY(ctx->lookback.ensure(2 * lb_region + 16));
        B2S_TRY(ctx->plan.ensure(2 * sizeof(RadixPlan)));
        own = {ctx->alt_keys.ptr, static_cast<uint32_t*>(ctx->alt_vals.ptr), ctx->lookback.ptr,
               static_cast<RadixCounters*>(ctx->hist.ptr), static_cast<RadixPlan*>(ctx->plan.ptr)};
        sc = &own;
    }
    const RadixPlan* cond = top_mode == 2 ? sc->plan : nullptr;
    RadixPlan* plan = sc->plan + (top_mode == 2 ? 1 : 0);
    RadixCounters* ctr = sc->ctr;
    const bool wide = !narrow_lookback_words(n, lookback_tile(n, (int)sizeof(U), VALS));
    ctx->ev_hist0 = record(ctx);
    B2S_CUDA(cudaMemsetAsync(ctr, 0, sizeof(RadixCounters), ctx->stream));
    // 4-byte keys past a few million: every digit histogram up front. 8-byte
    // keys only with B2S_ALL_HIST=2: measured for 2^28 u64 + u32 payload, the
    // 8-digit prologue takes 0.57 ms vs 0.37 for the digit-0 one, and the
    // pairs' passes gain nothing from skipping the in-pass count (1.96 ms)
    const bool all_hist = n >= kAllHistMinKeys && all_hist_mode() >= (sizeof(U) == 4 ? 1 : 2);
    if (all_hist) {
        static DeviceOnce once;
        B2S_TRY(once_per_device(once, ctx->device, [&]() -> b2s_status {
            B2S_CUDA(cudaFuncSetAttribute(radix_prologue_all_kernel<U>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAllHistSmem));
            return B2S_OK;
        }));
        const uint64_t want = (n / (16 / sizeof(U)) + kAllHistThreads * 4 - 1) / (kAllHistThreads * 4);
        const int grid = (int)std::min<uint64_t>(std::max<uint64_t>(want, 1), (uint64_t)ctx->num_sms);
        // look-back region 0 serves the first pass, which a keys-only sort
        // runs without look-back (tickets): nothing to zero then
        const size_t zero16 = (!VALS && B2S_TICKET_FIRST) ? 0 : (lb_region + 15) / 16;
        radix_prologue_all_kernel<U><<<grid, kAllHistThreads, kAllHistSmem, ctx->stream>>>(
            static_cast<const U*>(kin), n, ctr, static_cast<uint4*>(sc->lookback), zero16, top_xor, cond);
        B2S_LAUNCHED();
    } else {
        const int threads = 512;
        uint64_t want = (n / (16 / sizeof(U)) + threads - 1) / threads;
        int grid = (int)std::min<uint64_t>(std::max<uint64_t>(want, 1),
                                           (uint64_t)ctx->num_sms * kPrologueMinBlocks<U>);
        if (top_mode == 1 && sizeof(U) == 8)
            radix_prologue_kernel<U, true><<<grid, threads, 0, ctx->stream>>>(
                static_cast<const U*>(kin), n, ctr, static_cast<uint4*>(sc->lookback),
                (lb_region + 15) / 16, cond);
        else
            radix_prologue_kernel<U><<<grid, threads, 0, ctx->stream>>>(
                static_cast<const U*>(kin), n, ctr, static_cast<uint4*>(sc->lookback),
                (lb_region + 15) / 16, cond);
        B2S_LAUNCHED();
    }
    if (n >= kOrderCheckMinKeys && top_mode != 2) {
        const U flip = is_signed ? (U)1 << (8 * sizeof(U) - 1) : (U)0;
        const int grid = (int)std::min<uint64_t>((n / (16 / sizeof(U)) + 511) / 512, (uint64_t)ctx->num_sms * 4);
        radix_order_check_kernel<U><<<std::max(grid, 1), 512, 0, ctx->stream>>>(static_cast<const U*>(kin), n, ctr, flip);
        B2S_LAUNCHED();
    }
    radix_plan_kernel<<<1, 32, 0, ctx->stream>>>(plan, ctr, NP, n, top_xor, kin, kout,
                                                 sc->alt_keys, vin, vout, sc->alt_vals, all_hist ? 1 : 0,
                                                 top_mode, cond);
    B2S_LAUNCHED();
    if (n > 0 && !all_hist) {  // the all-digit prologue needs no recount
        int grid = (int)std::min<uint64_t>((n + 511) / 512, (uint64_t)ctx->num_sms * 4);
        radix_fallback_hist_kernel<U><<<grid, 512, 0, ctx->stream>>>(plan, static_cast<const U*>(kin),
                                                                     n, ctr);
        B2S_LAUNCHED();
    }
    ctx->ev_hist1 = record(ctx);
    ctx->last_passes_possible = NP;

    if (n > 0) {
        if (wide)
            B2S_TRY((launch_passes<U, VALS, unsigned long long>(ctx, plan, ctr, n, sc->lookback)));
        else
            B2S_TRY((launch_passes<U, VALS, uint32_t>(ctx, plan, ctr, n, sc->lookback)));
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

// Checks the property the atomic ranking relies on: lanes of one warp
// instruction adding to the same shared counter get old values in ascending
// lane order -- with the packed 16-bit counters and the inline-PTX atomics
// the ranking issues, also when some lanes are predicated off (the skewed
// pass's hot-digit lanes). Every warp keeps private counters; digit patterns
// run from one bin (all lanes collide) to 256 bins.
__global__ void probe_lane_order_kernel(int iters, unsigned long long* bad) {
    __shared__ uint32_t cnt[8][kRadix / 2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    unsigned long long nb = 0;
    for (int it = 0; it < iters; ++it) {
        for (int i = lane; i < kRadix / 2; i += 32) cnt[warp][i] = 0;
        __syncwarp();
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        const uint32_t bins = 1u << (it % 9);
        const uint32_t d = (x >> 8) % bins;
        const uint32_t sh16 = 16 * (d & 1);
        // odd iterations: about one lane in four sits out
        const bool on = (it & 1) == 0 || (x & 3) != 0;
        const uint32_t a = smem_addr(&cnt[warp][d >> 1]);
        const uint32_t r = (atom_add_shared_if(on, a, 1u << sh16) >> sh16) & 0xFFFFu;
        const uint32_t peers = match_digit<8>(d) & __ballot_sync(0xffffffffu, on);
        nb += on && (r != (uint32_t)__popc(peers & lt));
        __syncwarp();
    }
    if (nb) atomicAdd(bad, nb);
}

}  // namespace

b2s_status probe_lane_order(b2s_ctx* ctx, bool* ok) {
    *ok = false;
    const char* e = getenv("B2S_RANK");
    if (e && std::string(e) == "ballot") return B2S_OK;  // forced off
    B2S_TRY(ctx->misc.ensure(64));
    unsigned long long* bad = static_cast<unsigned long long*>(ctx->misc.ptr);
    B2S_CUDA(cudaMemsetAsync(bad, 0, 8, ctx->stream));
    probe_lane_order_kernel<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(288, bad);
    B2S_LAUNCHED();
    unsigned long long h = 1;
    B2S_CUDA(cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
    B2S_CUDA(cudaStreamSynchronize(ctx->stream));
    *ok = h == 0;
    return B2S_OK;
}

#ifdef B2S_PHASE_PROFILE
extern "C" int b2s_debug_phase_cycles(unsigned long long* out16, int reset) {
    cudaMemcpyFromSymbol(out16, b2s_phase_cycles, sizeof(b2s_phase_cycles));
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(b2s_phase_cycles, z, sizeof(z));
    }
    return 0;
}
#endif

size_t lookback_region_bytes(uint64_t n, int kbytes, bool vals) {
    const uint64_t tile = lookback_tile(n, kbytes, vals);
    const uint64_t ntiles = (n + tile - 1) / tile;
    return ntiles * kRadix * (narrow_lookback_words(n, tile) ? 4 : 8);
}

b2s_status radix_sort(b2s_ctx* ctx, b2s_dtype dtype, const void* kin, void* kout,
                      const uint32_t* vin, uint32_t* vout, uint64_t n, const SortScratch* sc) {
    const bool sgn = key_signed(dtype);
    const bool vals = vin != nullptr;
    // The pass plan's buffer chain treats keys and payload alike (in place or
    // not). Mixed aliasing -- keys in place with the payload out of place or
    // the reverse -- first copies the out-of-place array to its destination
    // and then sorts both in place.
    if (vals && n > 0 && (kin == kout) != (vin == vout)) {
        if (kin == kout) {
            B2S_CUDA(cudaMemcpyAsync(vout, vin, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
            vin = vout;
        } else {
            B2S_CUDA(cudaMemcpyAsync(kout, kin, n * (size_t)key_bytes(dtype), cudaMemcpyDeviceToDevice,
                                     ctx->stream));
            kin = kout;
        }
    }
    if (key_bytes(dtype) == 4) {
        return vals ? radix_sort_t<uint32_t, true>(ctx, sgn, kin, kout, vin, vout, n, sc)
                    : radix_sort_t<uint32_t, false>(ctx, sgn, kin, kout, vin, vout, n, sc);
    }
    using K = unsigned long long;
    // upper digits first (radix_plan_kernel decides on the device whether the
    // keys fit; if not, this first sort is the plain one and the rest no-ops)
    const bool top = sc == nullptr && n >= kTopFirstMinKeys && n <= kTopFirstMaxKeys && topfirst_enabled();
    if (!top) {
        return vals ? radix_sort_t<K, true>(ctx, sgn, kin, kout, vin, vout, n, sc)
                    : radix_sort_t<K, false>(ctx, sgn, kin, kout, vin, vout, n, sc);
    }
    B2S_TRY(vals ? (radix_sort_t<K, true>(ctx, sgn, kin, kout, vin, vout, n, nullptr, 1))
                 : (radix_sort_t<K, false>(ctx, sgn, kin, kout, vin, vout, n, nullptr, 1)));
    RadixPlan* plan = static_cast<RadixPlan*>(ctx->plan.ptr);
    {
        const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->num_sms * 16);
        if (vals)
            topfirst_fixup_kernel<true><<<grid, 256, 0, ctx->stream>>>(plan, static_cast<K*>(kout), vout, n);
        else
            topfirst_fixup_kernel<false><<<grid, 256, 0, ctx->stream>>>(plan, static_cast<K*>(kout), vout, n);
        B2S_LAUNCHED();
    }
    // the conditional full sort, in place; the timing keeps the first sort's
    // events (its passes are the ones that normally run) and ends after it
    const bool timing = ctx->timing;
    const int e_h0 = ctx->ev_hist0, e_h1 = ctx->ev_hist1;
    int e_pass[kMaxSlots + 1];
    for (int s = 0; s <= kMaxSlots; ++s) e_pass[s] = ctx->ev_pass[s];
    ctx->timing = false;
    const b2s_status st = vals ? radix_sort_t<K, true>(ctx, sgn, kout, kout, vout, vout, n, nullptr, 2)
                               : radix_sort_t<K, false>(ctx, sgn, kout, kout, vout, vout, n, nullptr, 2);
    ctx->timing = timing;
    ctx->ev_hist0 = e_h0;
    ctx->ev_hist1 = e_h1;
    for (int s = 0; s <= kMaxSlots; ++s) ctx->ev_pass[s] = e_pass[s];
    ctx->ev_copy1 = record(ctx);
    return st;
}

}  // namespace b2s
