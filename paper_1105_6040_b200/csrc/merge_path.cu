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

constexpr int kMergeThreads = 256;
template <typename T>
struct MergeItems {
#ifdef B2S_MERGE_ITEMS
    static constexpr int value = sizeof(T) == 4 ? B2S_MERGE_ITEMS : B2S_MERGE_ITEMS64;
#else
    // odd: conflict-free restaging. u32 2-way round of 2^28 keys: 11 items
    // 0.607 ms, 15: 0.572, 19: 0.555, 23: 0.558; u64 round of 2^27: 7 items
    // 0.562 ms, 11: 0.485, 15: 0.459 (19 overflows 48 KB with a payload)
    static constexpr int value = sizeof(T) == 4 ? 19 : 15;
#endif
};

// Merges output positions [out_lo, out_hi) of merge(A, B) into out[0 ..).
// Used both for full merges (out_lo = 0) and for merge_split's kept half.
// (A persistent variant that streams tile t + gridDim.x into a second buffer
// while tile t merges measured slower: 2.21 vs 1.78 ms for 8 runs of 2^25.)
template <typename T, bool VALS>
__global__ void __launch_bounds__(kMergeThreads) merge_tile_kernel(
    const T* __restrict__ a, const uint32_t* __restrict__ va, uint64_t na,
    const T* __restrict__ b, const uint32_t* __restrict__ vb, uint64_t nb,
    const uint64_t* __restrict__ parts, uint64_t out_lo, uint64_t out_hi, T* __restrict__ out,
    uint32_t* __restrict__ vout) {
    constexpr int ITEMS = MergeItems<T>::value;
    constexpr int TILE = kMergeThreads * ITEMS;
    __shared__ T s_k[TILE + 1];  // +1: the merge loop may read one past the end
    __shared__ uint32_t s_v[VALS ? TILE : 1];

    const uint64_t t = blockIdx.x;
    const uint64_t d0 = out_lo + t * TILE;
    const uint64_t d1 = std::min<uint64_t>(d0 + TILE, out_hi);
    const uint64_t a0 = parts[t], a1 = parts[t + 1];
    const uint64_t b0 = d0 - a0;
    const uint32_t la = (uint32_t)(a1 - a0), cnt = (uint32_t)(d1 - d0), lb = cnt - la;

    // stage A's slice then B's with asynchronous copies (no registers held,
    // every copy of the tile in flight at once)
    for (uint32_t i = threadIdx.x; i < cnt; i += kMergeThreads) {
        cp_async_elem(&s_k[i], i < la ? a + a0 + i : b + b0 + (i - la));
        if constexpr (VALS) cp_async_elem(&s_v[i], i < la ? va + a0 + i : vb + b0 + (i - la));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    const uint32_t diag = std::min<uint32_t>(threadIdx.x * ITEMS, cnt);
    uint32_t ai = merge_path_smem(s_k, la, s_k + la, lb, diag);
    uint32_t bi = la + diag - ai;  // index into the staged B
    // the two heads live in registers: one shared load per output
    T ka = s_k[ai], kb = s_k[bi];
    T rk[ITEMS];
    uint32_t rv[VALS ? ITEMS : 1];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        if (diag + j < cnt) {
            const bool take_a = bi >= cnt || (ai < la && !(kb < ka));
            rk[j] = take_a ? ka : kb;
            if constexpr (VALS) rv[j] = s_v[take_a ? ai : bi];
            const uint32_t nxt = take_a ? ++ai : ++bi;
            const T kn = s_k[nxt];
            if (take_a) ka = kn;
            else kb = kn;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        if (diag + j < cnt) {
            s_k[threadIdx.x * ITEMS + j] = rk[j];
            if constexpr (VALS) s_v[threadIdx.x * ITEMS + j] = rv[j];
        }
    }
    __syncthreads();
    const uint64_t o = d0 - out_lo;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const uint32_t i = threadIdx.x + j * kMergeThreads;
        if (i < cnt) {
            __stcs(out + o + i, s_k[i]);
            if constexpr (VALS) __stcs(vout + o + i, s_v[i]);
        }
    }
}

template <typename T>
__global__ void copy_kernel(const T* __restrict__ s, T* __restrict__ d, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        d[i] = s[i];
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
// Single-pass k-way merge (k <= kMaxK), replacing ceil(log2 k) pairwise rounds.
//
// Every S-th element of every run is a boundary record (key, run, position).
// kmerge_bounds_kernel places each boundary exactly: its cut in every other run
// is a binary search (ties: lower runs' equal keys come first), its rank among
// all boundaries is the number of each run's boundaries before those cuts.
// Between two consecutive boundaries in that order each run contributes at
// most S elements, so a bucket holds <= k*S keys and fits in shared memory.
// kmerge_bucket_kernel loads each bucket's k sub-ranges with coalesced reads,
// merges them pairwise in shared memory (log2 k rounds, stable: ties to the
// lower run) and writes the bucket with coalesced stores at its output offset
// (the sum of its lower cuts). HBM traffic: one read + one write per key.

constexpr int kMaxK = 16;

template <typename T>
struct KRuns {
    const T* key[kMaxK];
    const uint32_t* val[kMaxK];
    uint64_t n[kMaxK];
    uint64_t nb_off[kMaxK + 1];  // prefix of boundaries per run
    int k;
    uint32_t S;                   // boundary stride
};

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

template <typename T>
__global__ void kmerge_bounds_kernel(const KRuns<T> R, uint64_t* __restrict__ cuts) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= R.nb_off[R.k]) return;
    int r = 0;
    while (q >= R.nb_off[r + 1]) ++r;
    const uint64_t j = q - R.nb_off[r];
    const uint64_t pos = (j + 1) * R.S - 1;
    const T v = R.key[r][pos];
    uint64_t c[kMaxK];
    uint64_t rank = j;
    for (int r2 = 0; r2 < R.k; ++r2) {
        uint64_t cut;
        if (r2 == r) cut = pos + 1;
        else cut = bound_in(R.key[r2], R.n[r2], v, r2 < r);
        c[r2] = cut;
        if (r2 != r) rank += cut / R.S;
    }
    for (int r2 = 0; r2 < R.k; ++r2) cuts[rank * R.k + r2] = c[r2];
}

constexpr int kKThreads = 256;

template <typename T, bool VALS>
__global__ void __launch_bounds__(kKThreads) kmerge_bucket_kernel(const KRuns<T> R,
                                                                  const uint64_t* __restrict__ cuts,
                                                                  uint64_t nbuckets, uint32_t per_cta,
                                                                  uint32_t cap, T* __restrict__ out,
                                                                  uint32_t* __restrict__ vout) {
    extern __shared__ __align__(16) unsigned char smem[];
    T* kA = reinterpret_cast<T*>(smem);
    T* kB = kA + cap;
    uint32_t* vA = reinterpret_cast<uint32_t*>(kB + cap);
    uint32_t* vB = vA + (VALS ? cap : 0);
    __shared__ uint64_t s_lo[kMaxK];
    __shared__ uint32_t s_seg[kMaxK + 1];  // segment offsets inside the bucket
    __shared__ uint64_t s_out;
    const int k = R.k;
    const int tid = threadIdx.x;
    const uint64_t b0 = (uint64_t)blockIdx.x * per_cta;
    const uint64_t b1 = b0 + per_cta < nbuckets ? b0 + per_cta : nbuckets;
    for (uint64_t b = b0; b < b1; ++b) {
        if (tid == 0) {
            uint32_t acc = 0;
            uint64_t o = 0;
            for (int r = 0; r < k; ++r) {
                const uint64_t lo = b == 0 ? 0 : cuts[(b - 1) * k + r];
                const uint64_t hi = b + 1 == nbuckets ? R.n[r] : cuts[b * k + r];
                s_lo[r] = lo;
                s_seg[r] = acc;
                acc += (uint32_t)(hi - lo);
                o += lo;
            }
            s_seg[k] = acc;
            s_out = o;
        }
        __syncthreads();
        const uint32_t total = s_seg[k];
        // coalesced loads of the k sub-ranges, concatenated in run order
        for (int r = 0; r < k; ++r) {
            const uint32_t base = s_seg[r], len = s_seg[r + 1] - base;
            const T* src = R.key[r] + s_lo[r];
            for (uint32_t i = tid; i < len; i += kKThreads) kA[base + i] = src[i];
            if constexpr (VALS) {
                const uint32_t* vs = R.val[r] + s_lo[r];
                for (uint32_t i = tid; i < len; i += kKThreads) vA[base + i] = vs[i];
            }
        }
        __syncthreads();
        // pairwise rounds in shared memory; a pair keeps the position range of
        // its two segments, so segment offsets after a round are every other one
        T* ka = kA;
        T* kb = kB;
        uint32_t* va = vA;
        uint32_t* vb = vB;
        int nseg = k;
        int stride = 1;  // segments of this round start at s_seg[i * stride]
        while (nseg > 1) {
            constexpr int ITEMS = 8;
            for (uint32_t x0 = tid * ITEMS; x0 < total; x0 += kKThreads * ITEMS) {
                const uint32_t x1 = x0 + ITEMS < total ? x0 + ITEMS : total;
                uint32_t x = x0;
                while (x < x1) {
                    // the pair holding output position x
                    int pr = 0;
                    while (pr + 1 < (nseg + 1) / 2 && s_seg[min((pr + 1) * 2 * stride, k)] <= x) ++pr;
                    const uint32_t a0 = s_seg[min(pr * 2 * stride, k)];
                    const uint32_t a1 = s_seg[min(pr * 2 * stride + stride, k)];
                    const uint32_t e1 = s_seg[min(pr * 2 * stride + 2 * stride, k)];
                    const uint32_t la = a1 - a0, lb = e1 - a1;
                    const uint32_t diag = x - a0;
                    uint32_t ai = merge_path_smem(ka + a0, la, ka + a1, lb, diag);
                    uint32_t bi = diag - ai;
                    const uint32_t stop = x1 < e1 ? x1 : e1;
                    for (; x < stop; ++x) {
                        const bool take_a = bi >= lb || (ai < la && !(ka[a1 + bi] < ka[a0 + ai]));
                        const uint32_t src = take_a ? a0 + ai++ : a1 + bi++;
                        kb[x] = ka[src];
                        if constexpr (VALS) vb[x] = va[src];
                    }
                }
            }
            __syncthreads();
            T* t = ka;
            ka = kb;
            kb = t;
            uint32_t* tv = va;
            va = vb;
            vb = tv;
            nseg = (nseg + 1) / 2;
            stride *= 2;
        }
        const uint64_t o = s_out;
        for (uint32_t i = tid; i < total; i += kKThreads) {
            out[o + i] = ka[i];
            if constexpr (VALS) vout[o + i] = va[i];
        }
        __syncthreads();
    }
}

template <typename T>
b2s_status kway_single_pass(b2s_ctx* ctx, const void* const* runs, const uint32_t* const* vals,
                            const uint64_t* lens, int k, void* out, uint32_t* vout) {
    const bool with_vals = vout != nullptr;
    const size_t rec = sizeof(T) + (with_vals ? 4 : 0);
    // two buffers of `cap` records in <= 64 KB, cap = k * S with S a power of two
    uint32_t S = 1;
    const char* es = getenv("B2S_KWAY_SMEM_KB");
    const uint64_t budget = (uint64_t)(es ? atoi(es) : 64) * 1024;
    while ((uint64_t)2 * k * (S * 2) * rec <= budget) S *= 2;
    const uint32_t cap = (uint32_t)k * S;
    KRuns<T> R{};
    R.k = k;
    R.S = S;
    R.nb_off[0] = 0;
    uint64_t total = 0;
    for (int r = 0; r < k; ++r) {
        R.key[r] = static_cast<const T*>(runs[r]);
        R.val[r] = with_vals ? vals[r] : nullptr;
        R.n[r] = lens[r];
        R.nb_off[r + 1] = R.nb_off[r] + lens[r] / S;
        total += lens[r];
    }
    const uint64_t nb = R.nb_off[k];
    const uint64_t nbuckets = nb + 1;
    B2S_TRY(ctx->parts.ensure((nb * k + 1) * sizeof(uint64_t)));
    uint64_t* cuts = static_cast<uint64_t*>(ctx->parts.ptr);
    ctx->ev_merge0 = record(ctx);
    if (nb > 0) {
        kmerge_bounds_kernel<T><<<(unsigned)((nb + 255) / 256), 256, 0, ctx->stream>>>(R, cuts);
        B2S_LAUNCHED();
    }
    const size_t smem = (size_t)2 * cap * rec;
    auto kern = with_vals ? kmerge_bucket_kernel<T, true> : kmerge_bucket_kernel<T, false>;
    B2S_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint64_t want_ctas = (uint64_t)ctx->num_sms * 3 * 4;
    const uint32_t per_cta = (uint32_t)std::max<uint64_t>(1, (nbuckets + want_ctas - 1) / want_ctas);
    const unsigned grid = (unsigned)((nbuckets + per_cta - 1) / per_cta);
    kern<<<grid, kKThreads, smem, ctx->stream>>>(R, cuts, nbuckets, per_cta, cap,
                                                 static_cast<T*>(out), vout);
    B2S_LAUNCHED();
    ctx->ev_merge1 = record(ctx);
    ctx->last_merge_rounds = 1;
    (void)total;
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
        // 0: pairwise rounds (default: 3.5 TB/s per round on B200), 1: the
        // single-pass bucket merge (correct, but its in-shared-memory merge is
        // latency-bound at the occupancy its buffers allow: 3.5 ms vs 1.84 ms for
        // 8 runs of 2^25 keys -- kept for further work)
        const char* e = getenv("B2S_KWAY");
        m = e ? atoi(e) : 0;
    }
    return m;
}

template <typename T>
b2s_status kway_t(b2s_ctx* ctx, const void* const* runs, const uint32_t* const* vals,
                  const uint64_t* lens, int k, void* out, uint32_t* vout, void* tmp,
                  uint32_t* vtmp) {
    const bool with_vals = vout != nullptr;
    if (k > 2 && k <= kMaxK && kway_mode() == 1)
        return kway_single_pass<T>(ctx, runs, vals, lens, k, out, vout);
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
