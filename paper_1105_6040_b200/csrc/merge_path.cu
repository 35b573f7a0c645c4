// merge_path.cu -- stable merge-path merges for sm_100a.
//
// Replaces the root merge of the reference: the p odd-even merge_split phases
// and the rank-order gather (P/src/parallel_sort.cpp:59-134,217-248), whose
// result is the ascending concatenation of all blocks. kernels::merge_runs'
// tie rule (P/src/sort_core.cpp:46: ties take run_a) is kept everywhere, so a
// merge of runs 0..k-1 is stable with ties to the lower run index.
//
// 2-way merge of A and B into one output:
//   merge_partition_kernel  one thread per output tile boundary: merge-path
//                           binary search along the cross diagonal (log2 n
//                           probes, all boundaries in parallel).
//   merge_tile_kernel       one CTA per output tile: stage its A and B slices
//                           in shared memory with coalesced loads, each thread
//                           finds its own diagonal in shared memory and merges
//                           ITEMS outputs, results are restaged and written
//                           back with coalesced stores.
// k-way merge: ceil(log2 k) rounds of pairwise merges, ping-ponging between
// the output and a scratch buffer so the last round lands in the output.
// merge_split_padded: one merge-path tile pass restricted to the kept half.
#include <stdlib.h>

#include <algorithm>

#include "b2s_internal.cuh"

namespace b2s {
namespace {

// Number of A elements among the first `diag` outputs of merge(A, B) with
// ties taken from A first (a[i] <= b[j] -> a[i] goes first).
template <typename T>
__device__ __forceinline__ uint64_t merge_path(const T* a, uint64_t na, const T* b, uint64_t nb,
                                               uint64_t diag) {
    uint64_t lo = diag > nb ? diag - nb : 0;
    uint64_t hi = diag < na ? diag : na;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (!(b[diag - 1 - mid] < a[mid])) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename T>
__device__ __forceinline__ uint32_t merge_path_smem(const T* a, uint32_t na, const T* b,
                                                    uint32_t nb, uint32_t diag) {
    uint32_t lo = diag > nb ? diag - nb : 0;
    uint32_t hi = diag < na ? diag : na;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (!(b[diag - 1 - mid] < a[mid])) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// one element global -> shared, asynchronously (LDGSTS)
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    if constexpr (sizeof(T) == 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

#ifndef B2S_MERGE_ONE_LOAD
#define B2S_MERGE_ONE_LOAD 1  // 0: two predicated loads (u64 round of 2^27: 0.484 vs 0.463 ms)
#endif
constexpr int kMergeThreads = 256;
template <typename T>
struct MergeItems {
#ifdef B2S_MERGE_ITEMS
    static constexpr int value = sizeof(T) == 4 ? B2S_MERGE_ITEMS : B2S_MERGE_ITEMS64;
#else
    // odd: conflict-free restaging. u32 2-way round of 2^28 keys with the
    // shared-address merge step: 15 items 0.538 ms, 19: 0.505, 23: 0.481
    // (27 overflows 48 KB of static shared memory with a payload); u64 round
    // of 2^27: 11 items 0.458 ms, 15: 0.450 (round 1, index-based step: u32
    // 19 items 0.555 ms, u64 15 items 0.459)
    static constexpr int value = sizeof(T) == 4 ? 23 : 15;
#endif
};

// shared-memory record load / store by 32-bit shared address
template <typename T>
__device__ __forceinline__ T lds_rec(uint32_t a) {
    if constexpr (sizeof(T) == 4) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
        return (T)v;
    } else {
        unsigned long long v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
        return (T)v;
    }
}
template <typename T>
__device__ __forceinline__ void sts_rec(uint32_t a, T v) {
    if constexpr (sizeof(T) == 4)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"((uint32_t)v) : "memory");
    else
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"((unsigned long long)v) : "memory");
}

// 16 bytes global -> shared, asynchronously (both addresses 16-byte aligned)
__device__ __forceinline__ void cp_async_16(void* dst, const void* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

// Element phase of a global address within its 16-byte word.
template <typename T>
__device__ __forceinline__ uint32_t phase16(const T* p) {
    return (uint32_t)((reinterpret_cast<uintptr_t>(p) & 15u) / sizeof(T));
}

// Copies n elements src[0..n) to sdst[0..n) where sdst's address has the same
// 16-byte phase as src's: 16-byte cp.async for the aligned middle, single
// elements for the head and tail. All threads of the CTA take part.
template <typename T>
__device__ __forceinline__ void stage_slice(T* sdst, const T* src, uint32_t n) {
    constexpr uint32_t V = 16 / sizeof(T);
    const uint32_t ph = phase16(src);
    const uint32_t head = std::min<uint32_t>((V - ph) % V, n);
    const uint32_t nv = (n - head) / V;
    const uint32_t tail0 = head + nv * V;
    for (uint32_t v = threadIdx.x; v < nv; v += kMergeThreads)
        cp_async_16(sdst + head + v * V, src + head + v * V);
    const uint32_t t = threadIdx.x;
    if (t < head) cp_async_elem(sdst + t, src + t);
    else if (t >= V && t - V < n - tail0) cp_async_elem(sdst + tail0 + (t - V), src + tail0 + (t - V));
}

// Merges output positions [out_lo, out_hi) of merge(A, B) into out[0 ..).
// Used both for full merges (out_lo = 0) and for merge_split's kept half.
// The A and B slices are staged in shared memory at the same 16-byte phase as
// in global memory (vector copies), merged (heads in registers), restaged at
// the output's phase and written with 16-byte stores. (A persistent variant
// that streams tile t + gridDim.x into a second buffer while tile t merges
// measured slower: 2.21 vs 1.78 ms for 8 runs of 2^25.)
// Measured per 2-way round of 2^28 i32 keys: element-wise staging and stores
// 0.553 ms (53 instructions per output), vectorised 0.539 ms (48); the round
// is bound by shared-memory wavefronts (L1 79% busy: the merge loop's one
// load per output hits lanes' scattered heads) and issue (73%).
template <typename T, bool VALS>
__global__ void __launch_bounds__(kMergeThreads) merge_tile_kernel(
    const T* __restrict__ a, const uint32_t* __restrict__ va, uint64_t na,
    const T* __restrict__ b, const uint32_t* __restrict__ vb, uint64_t nb,
    const uint64_t* __restrict__ parts, uint64_t out_lo, uint64_t out_hi, T* __restrict__ out,
    uint32_t* __restrict__ vout) {
    constexpr int ITEMS = MergeItems<T>::value;
    constexpr int TILE = kMergeThreads * ITEMS;
    constexpr uint32_t V = 16 / sizeof(T);
    __shared__ __align__(16) T s_k[TILE + 3 * V + 1];  // two phase-aligned slices (+1: one read past the end)
    __shared__ __align__(16) uint32_t s_v[VALS ? TILE + 3 * 4 + 1 : 1];

    const uint64_t t = blockIdx.x;
    const uint64_t d0 = out_lo + t * TILE;
    const uint64_t d1 = std::min<uint64_t>(d0 + TILE, out_hi);
    const uint64_t a0 = parts[t], a1 = parts[t + 1];
    const uint64_t b0 = d0 - a0;
    const uint32_t la = (uint32_t)(a1 - a0), cnt = (uint32_t)(d1 - d0), lb = cnt - la;

    // A at s_k[pa ..), B at s_k[sb ..): each at its global 16-byte phase
    const uint32_t pa = phase16(a + a0);
    const uint32_t sb = (pa + la + V - 1) / V * V + phase16(b + b0);
    T* sa_ = s_k + pa;
    T* sb_ = s_k + sb;
    stage_slice(sa_, a + a0, la);
    stage_slice(sb_, b + b0, lb);
    uint32_t* sva = nullptr;
    uint32_t* svb = nullptr;
    if constexpr (VALS) {
        const uint32_t qa = phase16(va + a0);
        const uint32_t qb = (qa + la + 3) / 4 * 4 + phase16(vb + b0);
        sva = s_v + qa;
        svb = s_v + qb;
        stage_slice(sva, va + a0, la);
        stage_slice(svb, vb + b0, lb);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    const uint32_t diag = std::min<uint32_t>(threadIdx.x * ITEMS, cnt);
    uint32_t ai = merge_path_smem(sa_, la, sb_, lb, diag);
    uint32_t bi = diag - ai;
    T rk[ITEMS];
    uint32_t rv[VALS ? ITEMS : 1];
    if constexpr (!VALS) {
        // keys only: both heads and both read positions as shared byte
        // addresses in registers; per output one compare, one load of the
        // taken side's next record and selects (no index arithmetic)
        constexpr uint32_t SZ = sizeof(T);
        const uint32_t a_s = (uint32_t)__cvta_generic_to_shared(sa_);
        const uint32_t b_s = (uint32_t)__cvta_generic_to_shared(sb_);
        uint32_t qa = a_s + ai * SZ, qb = b_s + bi * SZ;
        const uint32_t ea = a_s + la * SZ, eb = b_s + lb * SZ;
        T ka = lds_rec<T>(qa), kb = lds_rec<T>(qb);
        auto step = [&](int j) {
            const bool ta = qa < ea && (qb >= eb || !(kb < ka));
            rk[j] = ta ? ka : kb;
            const uint32_t qn = (ta ? qa : qb) + SZ;
            const T v = lds_rec<T>(qn);
            qa = ta ? qn : qa;
            qb = ta ? qb : qn;
            ka = ta ? v : ka;
            kb = ta ? kb : v;
        };
        if (diag + ITEMS <= cnt) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) step(j);
        } else {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j)
                if (diag + j < cnt) step(j);
        }
    }
    // the two heads live in registers: one shared load per output
    T ka = sa_[ai], kb = sb_[bi];
#pragma unroll
    for (int j = 0; j < (VALS ? ITEMS : 0); ++j) {
        if (diag + j < cnt) {
            const bool take_a = bi >= lb || (ai < la && !(kb < ka));
            rk[j] = take_a ? ka : kb;
            if constexpr (VALS) rv[j] = take_a ? sva[ai] : svb[bi];
#if B2S_MERGE_ONE_LOAD
            // one shared load per step from the selected run (all lanes in
            // one instruction instead of two predicated half-warp loads)
            const T* np = take_a ? sa_ + ai + 1 : sb_ + bi + 1;
            ai += take_a ? 1u : 0u;
            bi += take_a ? 0u : 1u;
            const T kn = *np;
            ka = take_a ? kn : ka;
            kb = take_a ? kb : kn;
#else
            if (take_a) ka = sa_[++ai];
            else kb = sb_[++bi];
#endif
        }
    }
    __syncthreads();
    // restage at the output's 16-byte phase, then 16-byte stores
    const uint64_t o = d0 - out_lo;
    const uint32_t po = phase16(out + o);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        if (diag + j < cnt) s_k[po + threadIdx.x * ITEMS + j] = rk[j];
    }
    uint32_t pvo = 0;
    if constexpr (VALS) {
        pvo = phase16(vout + o);
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            if (diag + j < cnt) s_v[pvo + threadIdx.x * ITEMS + j] = rv[j];
        }
    }
    __syncthreads();
    {
        T* g = out + o;
        const uint32_t head = std::min<uint32_t>((V - po) % V, cnt);
        const uint32_t nv = (cnt - head) / V;
        const uint32_t tail0 = head + nv * V;
        for (uint32_t v = threadIdx.x; v < nv; v += kMergeThreads)
            __stcs(reinterpret_cast<uint4*>(g + head + v * V),
                   *reinterpret_cast<const uint4*>(s_k + po + head + v * V));
        const uint32_t th = threadIdx.x;
        if (th < head) __stcs(g + th, s_k[po + th]);
        else if (th >= V && th - V < cnt - tail0) __stcs(g + tail0 + (th - V), s_k[po + tail0 + (th - V)]);
    }
    if constexpr (VALS) {
        uint32_t* g = vout + o;
        const uint32_t head = std::min<uint32_t>((4 - pvo) % 4, cnt);
        const uint32_t nv = (cnt - head) / 4;
        const uint32_t tail0 = head + nv * 4;
        for (uint32_t v = threadIdx.x; v < nv; v += kMergeThreads)
            __stcs(reinterpret_cast<uint4*>(g + head + v * 4),
                   *reinterpret_cast<const uint4*>(s_v + pvo + head + v * 4));
        const uint32_t th = threadIdx.x;
        if (th < head) __stcs(g + th, s_v[pvo + th]);
        else if (th >= 4 && th - 4 < cnt - tail0) __stcs(g + tail0 + (th - 4), s_v[pvo + tail0 + (th - 4)]);
    }
}

template <typename T>
b2s_status copy_async(b2s_ctx* ctx, const T* s, T* d, uint64_t n) {
    if (n == 0 || s == d) return B2S_OK;
    B2S_CUDA(cudaMemcpyAsync(d, s, n * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
    return B2S_OK;
}

template <typename T>
__global__ void merge_partition_window_kernel(const T* __restrict__ a, uint64_t na,
                                              const T* __restrict__ b, uint64_t nb, uint64_t lo,
                                              uint64_t hi, uint64_t tile, uint64_t nparts,
                                              uint64_t* __restrict__ parts) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nparts) return;
    const uint64_t diag = std::min<uint64_t>(lo + i * tile, hi);
    parts[i] = merge_path(a, na, b, nb, diag);
}

// output positions [lo, hi) of merge(a, b) -> out[0, hi-lo)
template <typename T>
b2s_status merge2_window(b2s_ctx* ctx, const T* a, const uint32_t* va, uint64_t na, const T* b,
                         const uint32_t* vb, uint64_t nb, uint64_t lo, uint64_t hi, T* out,
                         uint32_t* vout) {
    constexpr int TILE = kMergeThreads * MergeItems<T>::value;
    if (hi <= lo) return B2S_OK;
    const uint64_t ntiles = (hi - lo + TILE - 1) / TILE;
    const uint64_t np = ntiles + 1;
    B2S_TRY(ctx->parts.ensure(np * sizeof(uint64_t)));
    uint64_t* parts = static_cast<uint64_t*>(ctx->parts.ptr);
    merge_partition_window_kernel<T><<<(unsigned)((np + 255) / 256), 256, 0, ctx->stream>>>(
        a, na, b, nb, lo, hi, TILE, np, parts);
    B2S_LAUNCHED();
    if (vout != nullptr)  // a run may be empty (null values) while the output has a payload
        merge_tile_kernel<T, true><<<(unsigned)ntiles, kMergeThreads, 0, ctx->stream>>>(
            a, va, na, b, vb, nb, parts, lo, hi, out, vout);
    else
        merge_tile_kernel<T, false><<<(unsigned)ntiles, kMergeThreads, 0, ctx->stream>>>(
            a, va, na, b, vb, nb, parts, lo, hi, out, vout);
    B2S_LAUNCHED();
    return B2S_OK;
}

// ---------------------------------------------------------------------------
// Grouped k-way merge (3 <= k <= kMaxK): one read and one write per key
// instead of ceil(log2 k) pairwise rounds.
//
// 1. Every S-th element of every run becomes a sample (key, run << 26 | chunk);
//    the samples are radix-sorted as pairs (stable: equal keys stay in run
//    order), which is the order of the samples in the merged output.
// 2. Every (T/S)-th sorted sample closes a group. Its cut in its own run is its
//    position + 1; in a lower run the elements <= its key come before it (ties
//    go to lower runs), in a higher run those < its key. A group then holds at
//    most S more elements per run than its T/S samples account for:
//    <= T + k*S keys (GroupSmem::CAP).
// 3. One CTA per group loads its k slices into shared memory (cp.async),
//    merges them pairwise in shared memory (log2 k rounds, ties to the lower
//    run, two heads in registers) and writes the group at its output offset
//    (the sum of its lower cuts) with coalesced stores.

constexpr int kMaxK = 16;
#ifndef B2S_KG_THREADS
#define B2S_KG_THREADS 256
#endif
constexpr int kKThreads = B2S_KG_THREADS;

#ifndef B2S_KG_CAP
#define B2S_KG_CAP 8192  // records per group (4-byte keys): two CTAs per SM
#endif
#ifndef B2S_KG_ITEMS
#define B2S_KG_ITEMS 29
#endif
template <typename T>
struct GroupCfg {
    static constexpr uint32_t S = sizeof(T) == 4 ? 256 : 128;              // sample stride
    static constexpr uint32_t CAP = sizeof(T) == 4 ? B2S_KG_CAP : 3200;    // records a group may hold
    // group target: with k runs a group then holds at most CAP records
    static constexpr uint32_t target(int k) { return CAP - (uint32_t)k * S; }
};

template <typename T>
struct KRuns {
    const T* key[kMaxK];
    const uint32_t* val[kMaxK];
    uint64_t n[kMaxK];
    uint64_t soff[kMaxK + 1];  // prefix of samples per run
    int k;
};

template <typename T>
__global__ void kmerge_samples_kernel(const KRuns<T> R, T* __restrict__ skeys,
                                      uint32_t* __restrict__ stags) {
    constexpr uint32_t S = GroupCfg<T>::S;
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= R.soff[R.k]) return;
    int r = 0;
    while (q >= R.soff[r + 1]) ++r;
    const uint64_t c = q - R.soff[r];
    skeys[q] = R.key[r][c * S + S - 1];
    stags[q] = ((uint32_t)r << 26) | (uint32_t)c;
}

template <typename T>
__device__ __forceinline__ uint64_t bound_in(const T* a, uint64_t n, T v, bool upper) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const T x = a[mid];
        if (x < v || (upper && !(v < x))) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// cuts[(g + 1) * k + r]: run r's cut at the end of group g; row 0 is zeros and
// the last row the run lengths
template <typename T>
__global__ void kmerge_cuts_kernel(const KRuns<T> R, const T* __restrict__ skeys,
                                   const uint32_t* __restrict__ stags, uint64_t ngroups,
                                   uint32_t per_group, uint64_t* __restrict__ cuts) {
    constexpr uint32_t S = GroupCfg<T>::S;
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int k = R.k;
    if (t >= (ngroups + 1) * k) return;
    const uint64_t g = t / k;  // boundary row
    const int r2 = (int)(t % k);
    uint64_t cut;
    if (g == 0) {
        cut = 0;
    } else if (g == ngroups) {
        cut = R.n[r2];
    } else {
        const uint64_t j = g * per_group - 1;  // closing sample of group g-1
        const T v = skeys[j];
        const int r = (int)(stags[j] >> 26);
        const uint64_t pos = (uint64_t)(stags[j] & ((1u << 26) - 1)) * S + S - 1;
        if (r2 == r) cut = pos + 1;
        else cut = bound_in(R.key[r2], R.n[r2], v, r2 < r);
    }
    cuts[g * k + r2] = cut;
}

// shared bytes of a group kernel for k runs: two buffers of cap records. The
// first buffer holds the k key slices each at its global 16-byte phase (up to
// V-1 records of padding per slice; the payload slices sit at the same
// indices of the value buffer), the output is restaged at its phase, and the
// merge reads one record past the end of a segment.
template <typename T, bool VALS>
constexpr uint32_t group_cap(int k) {
    return (GroupCfg<T>::CAP + (uint32_t)(2 * k + 2) * 4 + 4 + 3) / 4 * 4;
}
template <typename T, bool VALS>
constexpr size_t group_smem(uint32_t cap) {
    return 2 * (size_t)cap * sizeof(T) + (VALS ? 2 * (size_t)cap * 4 : 0);
}

// outputs per thread and merge round (odd: a warp's per-round output stores,
// ITEMS records apart, hit distinct banks)
template <typename T>
struct GroupItems {
    static constexpr int value = sizeof(T) == 4 ? B2S_KG_ITEMS : 13;
};

// Merge path on shared-memory segments given by byte address: the number of
// A records among the first `diag` outputs (ties to A).
template <typename T>
__device__ __forceinline__ uint32_t merge_path_sa(uint32_t a, uint32_t na, uint32_t b, uint32_t nb,
                                                  uint32_t diag) {
    uint32_t lo = diag > nb ? diag - nb : 0;
    uint32_t hi = diag < na ? diag : na;
    const uint32_t bd = b + (diag - 1) * (uint32_t)sizeof(T);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const bool a_first = !(lds_rec<T>(bd - mid * (uint32_t)sizeof(T)) < lds_rec<T>(a + mid * (uint32_t)sizeof(T)));
        lo = a_first ? mid + 1 : lo;
        hi = a_first ? hi : mid;
    }
    return lo;
}

// One group: its k slices are staged in shared memory (keys by 16-byte
// copies at their global phase, payloads element-wise at the same indices),
// merged pairwise in shared memory (ceil(log2 k) rounds, ties to the lower
// run; the last round writes at the output's 16-byte phase) and written with
// 16-byte stores. The merge step keeps both heads and both read positions
// (shared byte addresses) in registers: per output one compare, one store,
// one load of the taken side's next record and selects -- no index
// arithmetic. (The first version, index-based, issued 147 instructions per
// output for k = 8.)
template <typename T, bool VALS>
__global__ void __launch_bounds__(kKThreads) kmerge_group_kernel(const KRuns<T> R,
                                                                 const uint64_t* __restrict__ cuts,
                                                                 uint32_t cap, T* __restrict__ out,
                                                                 uint32_t* __restrict__ vout) {
    constexpr int ITEMS = GroupItems<T>::value;
    constexpr uint32_t V = 16 / sizeof(T);
    constexpr uint32_t SZ = sizeof(T);
    extern __shared__ __align__(16) unsigned char smem[];
    T* const kbase = reinterpret_cast<T*>(smem);
    uint32_t* const vbase = reinterpret_cast<uint32_t*>(smem + 2 * (size_t)cap * sizeof(T));
    __shared__ uint32_t s_seg[kMaxK + 1];  // output-space segments (prefix of lengths)
    __shared__ uint32_t s_kbeg[kMaxK];     // staged slices in buffer 0 (record index)
    __shared__ uint64_t s_lo[kMaxK];
    __shared__ uint64_t s_out;
    const int k = R.k;
    const int tid = threadIdx.x;
    const uint64_t g = blockIdx.x;
    if (tid < 32) {
        // lane r < k: run r's slice [lo, hi) of this group; its staged slot
        // spans roundup(phase + len, V) records, the keys start at its phase
        uint64_t lo = 0;
        uint32_t len = 0, ph = 0;
        if (tid < k) {
            lo = cuts[g * k + tid];
            len = (uint32_t)(cuts[(g + 1) * k + tid] - lo);
            ph = phase16(R.key[tid] + lo);
        }
        uint32_t acc = len, slot = (ph + len + V - 1) / V * V;
        uint64_t o = lo;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t a2 = __shfl_up_sync(0xffffffffu, acc, d);
            const uint32_t s2 = __shfl_up_sync(0xffffffffu, slot, d);
            if (tid >= d) {
                acc += a2;
                slot += s2;
            }
            o += __shfl_xor_sync(0xffffffffu, o, d);
        }
        if (tid < k) {
            s_lo[tid] = lo;
            s_seg[tid + 1] = acc;
            s_kbeg[tid] = slot - (ph + len + V - 1) / V * V + ph;
        }
        if (tid == 0) {
            s_seg[0] = 0;
            s_out = o;
        }
    }
    __syncthreads();
    const uint32_t total = s_seg[k];
    // warp w stages runs w, w + 8, ...: 16-byte copies of the aligned middle,
    // single records for the head and tail
    {
        const int lane = tid & 31;
        for (int r = tid >> 5; r < k; r += kKThreads / 32) {
            const uint32_t len = s_seg[r + 1] - s_seg[r];
            T* sd = kbase + s_kbeg[r];
            const T* src = R.key[r] + s_lo[r];
            const uint32_t head = min((V - phase16(src)) % V, len);
            const uint32_t nv = (len - head) / V;
            const uint32_t tail0 = head + nv * V;
            for (uint32_t v = lane; v < nv; v += 32) cp_async_16(sd + head + v * V, src + head + v * V);
            if ((uint32_t)lane < head) cp_async_elem(sd + lane, src + lane);
            else if ((uint32_t)lane >= V && lane - V < len - tail0)
                cp_async_elem(sd + tail0 + (lane - V), src + tail0 + (lane - V));
            if constexpr (VALS) {
                const uint32_t* vs = R.val[r] + s_lo[r];
                for (uint32_t i = lane; i < len; i += 32) cp_async_elem(vbase + s_kbeg[r] + i, vs + i);
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const uint64_t o = s_out;
    const uint32_t po = phase16(out + o);
    const uint32_t k0 = (uint32_t)__cvta_generic_to_shared(kbase);
    const uint32_t v0 = (uint32_t)__cvta_generic_to_shared(vbase);
    // payload address of the record at key address a (same record index)
    auto vaddr = [&](uint32_t a) -> uint32_t {
        return sizeof(T) == 4 ? a + (v0 - k0) : v0 + ((a - k0) >> 1);
    };
    // pairwise rounds in shared memory; after a round segment i spans the old
    // segments 2i and 2i+1
    int cur = 0;
    int m = k;
    bool first = true;
    while (m > 1) {
        const bool last = (m + 1) / 2 == 1;
        const uint32_t ks = k0 + (cur ? cap * SZ : 0u);
        const uint32_t kd = k0 + (cur ? 0u : cap * SZ) + (last ? po * SZ : 0u);
        // chunks of ITEMS outputs never straddle a pair: pair p owns chunks
        // [c(p), c(p+1)) with c(p) = sum of ceil(len / ITEMS) below it
        const int npairs = (m + 1) / 2;
        uint32_t nchunks = 0;
        for (int q = 0; q < npairs; ++q) nchunks += (s_seg[min(2 * q + 2, m)] - s_seg[2 * q] + ITEMS - 1) / ITEMS;
        // one merge chain per chunk: both heads and read positions as shared
        // byte addresses; the per-output step is a compare, a store, one load
        // of the taken side's next record and selects
        struct Chain {
            uint32_t pa, pb, ea, eb, od, n;
            T ka, kb;
        };
        auto open = [&](uint32_t c, Chain& h) {
            int p = 0;
            uint32_t c0 = 0;
            for (;;) {  // pair of chunk c
                const uint32_t n = (s_seg[min(2 * p + 2, m)] - s_seg[2 * p] + ITEMS - 1) / ITEMS;
                if (c < c0 + n) break;
                c0 += n;
                ++p;
            }
            // pair p: A = segment 2p, B = segment 2p+1 (empty past the end)
            const int ia = 2 * p, ib = 2 * p + 1;
            const uint32_t o0 = s_seg[ia];
            const uint32_t la = s_seg[ia + 1] - o0;
            const uint32_t lb = ib < m ? s_seg[ib + 1] - s_seg[ib] : 0u;
            const uint32_t a = ks + (first ? s_kbeg[ia] : o0) * SZ;
            const uint32_t b = ks + (first ? (ib < m ? s_kbeg[ib] : 0u) : o0 + la) * SZ;
            const uint32_t x = o0 + (c - c0) * ITEMS;
            const uint32_t diag = x - o0;
            const uint32_t ai = merge_path_sa<T>(a, la, b, lb, diag);
            h.pa = a + ai * SZ;
            h.pb = b + (diag - ai) * SZ;
            h.ea = a + la * SZ;
            h.eb = b + lb * SZ;
            h.ka = lds_rec<T>(h.pa);
            h.kb = lds_rec<T>(h.pb);
            h.n = min((uint32_t)ITEMS, o0 + la + lb - x);
            h.od = kd + x * SZ;
        };
        auto step = [&](Chain& h, uint32_t j) {
            const bool ta = h.pa < h.ea && (h.pb >= h.eb || !(h.kb < h.ka));
            const uint32_t pt = ta ? h.pa : h.pb;
            sts_rec<T>(h.od + j * SZ, ta ? h.ka : h.kb);
            if constexpr (VALS) sts_rec<uint32_t>(vaddr(h.od + j * SZ), lds_rec<uint32_t>(vaddr(pt)));
            const uint32_t pn = pt + SZ;
            const T v = lds_rec<T>(pn);
            h.pa = ta ? pn : h.pa;
            h.pb = ta ? h.pb : pn;
            h.ka = ta ? v : h.ka;
            h.kb = ta ? h.kb : v;
        };
        // two independent chains per thread (chunks c and c + kKThreads),
        // stepped in lockstep so one's shared-load latency hides behind the
        // other's compare and selects
        for (uint32_t c = tid; c < nchunks; c += 2 * kKThreads) {
            Chain h0, h1;
            open(c, h0);
            const bool two = c + kKThreads < nchunks;
            if (two) open(c + kKThreads, h1);
            if (two && h0.n == (uint32_t)ITEMS && h1.n == (uint32_t)ITEMS) {
#pragma unroll
                for (int j = 0; j < ITEMS; ++j) {
                    step(h0, j);
                    step(h1, j);
                }
            } else {
                for (uint32_t j = 0; j < h0.n; ++j) step(h0, j);
                if (two)
                    for (uint32_t j = 0; j < h1.n; ++j) step(h1, j);
            }
        }
        __syncthreads();
        if (tid == 0) {
            const int m2 = (m + 1) / 2;
            for (int i = 1; i <= m2; ++i) s_seg[i] = s_seg[min(2 * i, m)];
        }
        m = (m + 1) / 2;
        cur ^= 1;
        first = false;
        __syncthreads();
    }
    // the result sits at the output's 16-byte phase: 16-byte stores
    const T* kf = kbase + (cur ? cap : 0) + po;
    {
        T* gk = out + o;
        const uint32_t head = min((V - po) % V, total);
        const uint32_t nv = (total - head) / V;
        const uint32_t tail0 = head + nv * V;
        for (uint32_t v = tid; v < nv; v += kKThreads)
            __stcs(reinterpret_cast<uint4*>(gk + head + v * V), *reinterpret_cast<const uint4*>(kf + head + v * V));
        if ((uint32_t)tid < head) __stcs(gk + tid, kf[tid]);
        else if ((uint32_t)tid >= V && tid - V < total - tail0) __stcs(gk + tail0 + (tid - V), kf[tail0 + (tid - V)]);
    }
    if constexpr (VALS) {
        // payloads sit at the key records' indices (phase po in key records)
        const uint32_t* vf = vbase + (cur ? cap : 0) + po;
        uint32_t* gv = vout + o;
        for (uint32_t i = tid; i < total; i += kKThreads) __stcs(gv + i, vf[i]);
    }
}

template <typename T> constexpr b2s_dtype dtype_of();
template <> constexpr b2s_dtype dtype_of<int32_t>() { return B2S_I32; }
template <> constexpr b2s_dtype dtype_of<uint32_t>() { return B2S_U32; }
template <> constexpr b2s_dtype dtype_of<int64_t>() { return B2S_I64; }
template <> constexpr b2s_dtype dtype_of<unsigned long long>() { return B2S_U64; }

template <typename T, bool VALS>
b2s_status launch_groups(b2s_ctx* ctx, const KRuns<T>& R, const uint64_t* cuts, uint64_t ngroups,
                         T* out, uint32_t* vout) {
    auto kern = kmerge_group_kernel<T, VALS>;
    static DeviceOnce once;
    B2S_TRY(once_per_device(once, ctx->device, [&]() -> b2s_status {
        B2S_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)group_smem<T, VALS>(group_cap<T, VALS>(kMaxK))));
        return B2S_OK;
    }));
    const uint32_t cap = group_cap<T, VALS>(R.k);
    kern<<<(unsigned)ngroups, kKThreads, group_smem<T, VALS>(cap), ctx->stream>>>(R, cuts, cap, out, vout);
    B2S_LAUNCHED();
    return B2S_OK;
}

// sample tags hold a 26-bit chunk index
template <typename T>
bool kway_grouped_fits(const uint64_t* lens, int k) {
    for (int r = 0; r < k; ++r)
        if (lens[r] / GroupCfg<T>::S >= (1ull << 26)) return false;
    return true;
}

template <typename T>
b2s_status kway_grouped(b2s_ctx* ctx, const void* const* runs, const uint32_t* const* vals,
                        const uint64_t* lens, int k, void* out, uint32_t* vout) {
    constexpr uint32_t S = GroupCfg<T>::S;
    const uint32_t per_group = GroupCfg<T>::target(k) / S;
    const bool with_vals = vout != nullptr;
    KRuns<T> R{};
    R.k = k;
    R.soff[0] = 0;
    for (int r = 0; r < k; ++r) {
        R.key[r] = static_cast<const T*>(runs[r]);
        R.val[r] = with_vals ? vals[r] : nullptr;
        R.n[r] = lens[r];
        R.soff[r + 1] = R.soff[r] + lens[r] / S;
    }
    const uint64_t m = R.soff[k];
    const uint64_t ngroups = m / per_group + 1;
    // scratch: samples (in, sorted), tags (in, sorted), cuts
    const size_t sk = (m * sizeof(T) + 255) / 256 * 256, st = (m * 4 + 255) / 256 * 256;
    const size_t cb = (ngroups + 1) * k * sizeof(uint64_t);
    B2S_TRY(ctx->kmerge.ensure(2 * sk + 2 * st + cb + 256));
    char* base = static_cast<char*>(ctx->kmerge.ptr);
    T* s_in = reinterpret_cast<T*>(base);
    T* s_out = reinterpret_cast<T*>(base + sk);
    uint32_t* t_in = reinterpret_cast<uint32_t*>(base + 2 * sk);
    uint32_t* t_out = reinterpret_cast<uint32_t*>(base + 2 * sk + st);
    uint64_t* cuts = reinterpret_cast<uint64_t*>(base + 2 * sk + 2 * st);
    ctx->ev_merge0 = record(ctx);
    if (m > 0) {
        kmerge_samples_kernel<T><<<(unsigned)((m + 255) / 256), 256, 0, ctx->stream>>>(R, s_in, t_in);
        B2S_LAUNCHED();
        B2S_TRY(radix_sort(ctx, dtype_of<T>(), s_in, s_out, t_in, t_out, m));
    }
    const uint64_t nc = (ngroups + 1) * k;
    kmerge_cuts_kernel<T><<<(unsigned)((nc + 255) / 256), 256, 0, ctx->stream>>>(R, s_out, t_out, ngroups,
                                                                                per_group, cuts);
    B2S_LAUNCHED();
    if (with_vals)
        B2S_TRY((launch_groups<T, true>(ctx, R, cuts, ngroups, static_cast<T*>(out), vout)));
    else
        B2S_TRY((launch_groups<T, false>(ctx, R, cuts, ngroups, static_cast<T*>(out), vout)));
    ctx->ev_merge1 = record(ctx);
    ctx->last_merge_rounds = 1;
    return B2S_OK;
}

struct Run {
    const void* k;
    const uint32_t* v;
    uint64_t n;
};

int kway_mode() {
    static int m = -1;
    if (m < 0) {
        // -1 (default): the grouped single-pass merge for 4-byte keys,
        // 5 <= k <= 8 and n >= 2^22, pairwise rounds otherwise; 0: always
        // pairwise; 1: grouped whenever it applies. The grouped merge reads
        // and writes every key once, but its rounds in shared memory are
        // bound by the merge step's dependency chain and the per-group
        // barriers, not HBM. Measured per 2^28 i32 keys (pairwise / grouped):
        // k=3 0.901 / 1.064 ms, k=4 0.961 / 0.963, k=8 1.501 / 1.388, k=16
        // 2.141 / 2.313; per 2^27 u64 (pairwise): k=2 0.450, k=4 0.921, k=8
        // 1.441, k=16 2.065 (grouped 1.428 at k=8, slower elsewhere).
        const char* e = getenv("B2S_KWAY");
        m = e ? atoi(e) : -1;
    }
    return m;
}

template <typename T>
b2s_status kway_t(b2s_ctx* ctx, const void* const* runs, const uint32_t* const* vals,
                  const uint64_t* lens, int k, void* out, uint32_t* vout, void* tmp,
                  uint32_t* vtmp) {
    const bool with_vals = vout != nullptr;
    const int mode = kway_mode();
    uint64_t n_all = 0;
    for (int i = 0; i < k; ++i) n_all += lens[i];
    // small merges are bound by their chain of launches: the grouped one's
    // sample sort adds a dozen (cfg1, 4 runs of 2^18: 0.112 vs 0.09 ms)
    const bool grouped = mode == 1 || (mode < 0 && sizeof(T) == 4 && k >= 5 && k <= 8 && n_all >= (1ull << 22));
    if (k > 2 && k <= kMaxK && grouped && kway_grouped_fits<T>(lens, k))
        return kway_grouped<T>(ctx, runs, vals, lens, k, out, vout);
    std::vector<Run> cur;
    uint64_t total = 0;
    for (int i = 0; i < k; ++i) {
        cur.push_back({runs[i], with_vals ? vals[i] : nullptr, lens[i]});
        total += lens[i];
    }
    int rounds = 0;
    while ((1 << rounds) < k) ++rounds;
    ctx->last_merge_rounds = rounds;
    ctx->ev_merge0 = record(ctx);
    if (k == 1) {
        B2S_TRY(copy_async<T>(ctx, static_cast<const T*>(cur[0].k), static_cast<T*>(out), total));
        if (with_vals) B2S_TRY(copy_async<uint32_t>(ctx, cur[0].v, vout, total));
    }
    for (int r = 0; r < rounds; ++r) {
        const bool to_out = ((rounds - 1 - r) % 2) == 0;
        T* dst = static_cast<T*>(to_out ? out : tmp);
        uint32_t* vdst = with_vals ? (to_out ? vout : vtmp) : nullptr;
        std::vector<Run> nxt;
        uint64_t off = 0;
        for (size_t i = 0; i < cur.size(); i += 2) {
            if (i + 1 < cur.size()) {
                const Run& A = cur[i];
                const Run& B = cur[i + 1];
                B2S_TRY(merge2_window<T>(ctx, static_cast<const T*>(A.k), A.v, A.n,
                                         static_cast<const T*>(B.k), B.v, B.n, 0, A.n + B.n,
                                         dst + off, vdst ? vdst + off : nullptr));
                nxt.push_back({dst + off, vdst ? vdst + off : nullptr, A.n + B.n});
                off += A.n + B.n;
            } else {
                // odd run out: move it into this round's buffer so no later round
                // reads a buffer it is writing
                const Run& A = cur[i];
                B2S_TRY(copy_async<T>(ctx, static_cast<const T*>(A.k), dst + off, A.n));
                if (vdst) B2S_TRY(copy_async<uint32_t>(ctx, A.v, vdst + off, A.n));
                nxt.push_back({dst + off, vdst ? vdst + off : nullptr, A.n});
                off += A.n;
            }
        }
        cur.swap(nxt);
    }
    ctx->ev_merge1 = record(ctx);
    return B2S_OK;
}

template <typename T>
b2s_status merge_split_t(b2s_ctx* ctx, const void* mine, uint64_t nm, uint64_t mv,
                         const void* theirs, uint64_t nt, uint64_t tv, int keep_high, void* out,
                         uint64_t* out_n, uint64_t* out_v) {
    // merge_split_padded, P/src/parallel_sort.cpp:115-134. Low side: the
    // lowest min(width, reals) of merge(mine, theirs) with ties to mine
    // (merge_take_low :74). High side: the highest `width - virtuals`, filled
    // from the back taking theirs on ties (merge_take_high :97) -- the same
    // sequence as the top of merge(mine, theirs) with ties to mine.
    const uint64_t width = nm + mv;
    const uint64_t reals = nm + nt;
    if (!keep_high) {
        const uint64_t take = std::min(width, reals);
        *out_n = take;
        *out_v = width - take;
        return merge2_window<T>(ctx, static_cast<const T*>(mine), nullptr, nm,
                                static_cast<const T*>(theirs), nullptr, nt, 0, take,
                                static_cast<T*>(out), nullptr);
    }
    const uint64_t virt = std::min(width, mv + tv);
    const uint64_t take = width - virt;
    *out_n = take;
    *out_v = virt;
    return merge2_window<T>(ctx, static_cast<const T*>(mine), nullptr, nm,
                            static_cast<const T*>(theirs), nullptr, nt, reals - take, reals,
                            static_cast<T*>(out), nullptr);
}

}  // namespace

b2s_status kway_merge(b2s_ctx* ctx, b2s_dtype dtype, const void* const* runs,
                      const uint32_t* const* vals, const uint64_t* lens, int k, void* out,
                      uint32_t* vout, void* tmp, uint32_t* vtmp) {
    switch (dtype) {
        case B2S_I32: return kway_t<int32_t>(ctx, runs, vals, lens, k, out, vout, tmp, vtmp);
        case B2S_U32: return kway_t<uint32_t>(ctx, runs, vals, lens, k, out, vout, tmp, vtmp);
        case B2S_I64: return kway_t<int64_t>(ctx, runs, vals, lens, k, out, vout, tmp, vtmp);
        case B2S_U64:
            return kway_t<unsigned long long>(ctx, runs, vals, lens, k, out, vout, tmp, vtmp);
    }
    return set_error(B2S_EINVAL, "bad dtype");
}

b2s_status merge_split_padded(b2s_ctx* ctx, b2s_dtype dtype, const void* mine, uint64_t nm,
                              uint64_t mv, const void* theirs, uint64_t nt, uint64_t tv,
                              int keep_high, void* out, uint64_t* out_n, uint64_t* out_v) {
    switch (dtype) {
        case B2S_I32:
            return merge_split_t<int32_t>(ctx, mine, nm, mv, theirs, nt, tv, keep_high, out,
                                          out_n, out_v);
        case B2S_U32:
            return merge_split_t<uint32_t>(ctx, mine, nm, mv, theirs, nt, tv, keep_high, out,
                                           out_n, out_v);
        case B2S_I64:
            return merge_split_t<int64_t>(ctx, mine, nm, mv, theirs, nt, tv, keep_high, out,
                                          out_n, out_v);
        case B2S_U64:
            return merge_split_t<unsigned long long>(ctx, mine, nm, mv, theirs, nt, tv,
                                                     keep_high, out, out_n, out_v);
    }
    return set_error(B2S_EINVAL, "bad dtype");
}

}  // namespace b2s
