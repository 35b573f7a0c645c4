/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's partitioned-sort path
 * (/root/reference/proj, "sortbench"), used as the parity checker for the
 * B200 kernels. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the timed CPU baseline -- never as a product code path.
 *
 * Parity of this restatement is pinned against the reference itself:
 * oracle/build_ref.sh compiles the reference sources into oracle/_ref and
 * tests/golden/make_golden.py records its outputs; tests/test_oracle.py checks
 * this file against those fixtures.
 *
 * Every function names the reference lines it restates.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_GAMMA 0x9E3779B97F4A7C15ULL

/* splitmix64 finaliser, as in bench::gen_data (P/src/bench.cpp:62-67). */
static inline uint64_t orc_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* bench::gen_data(n, seed) -- P/src/bench.cpp:57-71. Element i is
 * mix(seed + (i+1)*gamma) reinterpreted as int64. `first` lets a caller
 * generate a window [first, first+n) of the same stream (shards). */
void orc_gen_data(uint64_t first, uint64_t n, uint64_t seed, int64_t* out) {
    uint64_t x = seed + first * ORC_GAMMA;
    for (uint64_t i = 0; i < n; ++i) {
        x += ORC_GAMMA;
        out[i] = (int64_t)orc_mix(x);
    }
}

/* parallel::plan_partition(n, p) -- P/src/parallel_sort.cpp:26-38: the first
 * n mod p ranks get one extra element. Returns -1 for p < 1 (ConfigError). */
int orc_plan_partition(uint64_t n, int p, uint64_t* sizes) {
    if (p < 1) return -1;
    const uint64_t base = n / (uint64_t)p;
    const uint64_t extra = n % (uint64_t)p;
    for (int r = 0; r < p; ++r) sizes[r] = base + ((uint64_t)r < extra ? 1u : 0u);
    return 0;
}

/* parallel::build_schedule(p) -- P/src/parallel_sort.cpp:40-55. partners is
 * a p*p row-major [phase][rank] table, -1 when the rank idles. */
int orc_build_schedule(int p, int* partners) {
    if (p < 1) return -1;
    for (int phase = 0; phase < p; ++phase) {
        int* row = partners + (size_t)phase * (size_t)p;
        for (int r = 0; r < p; ++r) row[r] = -1;
        for (int r = (phase % 2 == 0) ? 0 : 1; r + 1 < p; r += 2) {
            row[r] = r + 1;
            row[r + 1] = r;
        }
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Sequential kernels, generic over the key type. The reference only has
 * int64 (P/include/sortbench/element.hpp:10); the u32/i32/u64 versions are the
 * widened restatement SURVEY.md section 8(c) prescribes, with the same tie rule.
 */

/* kernels::merge_runs -- P/src/sort_core.cpp:38-62. Stable: ties take run_a. */
#define ORC_DEFINE_MERGE_RUNS(NAME, T)                                          \
    void NAME(const T* a, uint64_t na, const T* b, uint64_t nb, T* out) {       \
        uint64_t i = 0, j = 0, k = 0;                                           \
        while (i < na && j < nb) out[k++] = (a[i] <= b[j]) ? a[i++] : b[j++];   \
        while (i < na) out[k++] = a[i++];                                       \
        while (j < nb) out[k++] = b[j++];                                       \
    }

ORC_DEFINE_MERGE_RUNS(orc_merge_runs_i64, int64_t)
ORC_DEFINE_MERGE_RUNS(orc_merge_runs_u64, uint64_t)
ORC_DEFINE_MERGE_RUNS(orc_merge_runs_i32, int32_t)
ORC_DEFINE_MERGE_RUNS(orc_merge_runs_u32, uint32_t)

/* kernels::merge_sort + merge_in_place -- P/src/sort_core.cpp:66-106:
 * top-down, inclusive bounds [first, last], one scratch buffer, ties take the
 * lower half. first > last (and first == last) return immediately. The
 * recursion is restated with an explicit depth-first order identical to the
 * reference's (mid = (first+last)/2). */
#define ORC_DEFINE_MERGE_SORT(NAME, T)                                          \
    static void NAME##_merge(T* blk, int64_t first, int64_t mid, int64_t last,  \
                             T* scratch) {                                      \
        int64_t i = first, j = mid + 1, k = first;                              \
        while (i <= mid && j <= last)                                           \
            scratch[k++] = (blk[i] <= blk[j]) ? blk[i++] : blk[j++];            \
        while (i <= mid) scratch[k++] = blk[i++];                               \
        while (j <= last) scratch[k++] = blk[j++];                              \
        memcpy(blk + first, scratch + first, (size_t)(last - first + 1) * sizeof(T)); \
    }                                                                           \
    void NAME(T* blk, int64_t first, int64_t last, T* scratch) {                \
        if (first >= last) return;                                              \
        const int64_t mid = (first + last) / 2;                                 \
        NAME(blk, first, mid, scratch);                                         \
        NAME(blk, mid + 1, last, scratch);                                      \
        NAME##_merge(blk, first, mid, last, scratch);                           \
    }

ORC_DEFINE_MERGE_SORT(orc_merge_sort_i64, int64_t)
ORC_DEFINE_MERGE_SORT(orc_merge_sort_u64, uint64_t)
ORC_DEFINE_MERGE_SORT(orc_merge_sort_i32, int32_t)
ORC_DEFINE_MERGE_SORT(orc_merge_sort_u32, uint32_t)

/* Stable key/value sort: the reference has no payload (F1); the restatement is
 * merge_sort's stable tie rule (P/src/sort_core.cpp:77) applied to (key, val)
 * records ordered by key only -- i.e. std::stable_sort by key. */
#define ORC_DEFINE_KV_SORT(NAME, K)                                             \
    static void NAME##_rec(K* k, uint32_t* v, int64_t first, int64_t last,      \
                           K* sk, uint32_t* sv) {                               \
        if (first >= last) return;                                              \
        const int64_t mid = (first + last) / 2;                                 \
        NAME##_rec(k, v, first, mid, sk, sv);                                   \
        NAME##_rec(k, v, mid + 1, last, sk, sv);                                \
        int64_t i = first, j = mid + 1, o = first;                              \
        while (i <= mid && j <= last) {                                         \
            if (k[i] <= k[j]) { sk[o] = k[i]; sv[o++] = v[i++]; }               \
            else { sk[o] = k[j]; sv[o++] = v[j++]; }                            \
        }                                                                       \
        while (i <= mid) { sk[o] = k[i]; sv[o++] = v[i++]; }                    \
        while (j <= last) { sk[o] = k[j]; sv[o++] = v[j++]; }                   \
        memcpy(k + first, sk + first, (size_t)(last - first + 1) * sizeof(K));  \
        memcpy(v + first, sv + first, (size_t)(last - first + 1) * sizeof(uint32_t)); \
    }                                                                           \
    int NAME(K* keys, uint32_t* vals, uint64_t n) {                             \
        if (n < 2) return 0;                                                    \
        K* sk = (K*)malloc(n * sizeof(K));                                      \
        uint32_t* sv = (uint32_t*)malloc(n * sizeof(uint32_t));                 \
        if (!sk || !sv) { free(sk); free(sv); return -1; }                      \
        NAME##_rec(keys, vals, 0, (int64_t)n - 1, sk, sv);                      \
        free(sk); free(sv);                                                     \
        return 0;                                                               \
    }

ORC_DEFINE_KV_SORT(orc_stable_sort_kv_u64, uint64_t)
ORC_DEFINE_KV_SORT(orc_stable_sort_kv_u32, uint32_t)
ORC_DEFINE_KV_SORT(orc_stable_sort_kv_i32, int32_t)
ORC_DEFINE_KV_SORT(orc_stable_sort_kv_i64, int64_t)

/* Whole-array sorts through merge_sort (the reference's `merge` kernel,
 * P/src/parallel_sort.cpp:143-148) for each key width. */
#define ORC_DEFINE_SORT(NAME, MS, T)                                            \
    int NAME(T* keys, uint64_t n) {                                             \
        if (n < 2) return 0;                                                    \
        T* scratch = (T*)malloc(n * sizeof(T));                                 \
        if (!scratch) return -1;                                                \
        MS(keys, 0, (int64_t)n - 1, scratch);                                   \
        free(scratch);                                                          \
        return 0;                                                               \
    }

ORC_DEFINE_SORT(orc_sort_i64, orc_merge_sort_i64, int64_t)
ORC_DEFINE_SORT(orc_sort_u64, orc_merge_sort_u64, uint64_t)
ORC_DEFINE_SORT(orc_sort_i32, orc_merge_sort_i32, int32_t)
ORC_DEFINE_SORT(orc_sort_u32, orc_merge_sort_u32, uint32_t)

/* ---------------------------------------------------------------------------
 * Odd-even merge-split, P/src/parallel_sort.cpp:59-134.
 */

/* merge_take_low -- :60-80: the lowest `take` of mine U theirs, ties to mine. */
static void orc_take_low(const int64_t* mine, uint64_t nm, const int64_t* theirs,
                         uint64_t nt, uint64_t take, int64_t* out) {
    uint64_t i = 0, j = 0;
    for (uint64_t k = 0; k < take; ++k) {
        int take_mine;
        if (i >= nm) take_mine = 0;
        else if (j >= nt) take_mine = 1;
        else take_mine = mine[i] <= theirs[j];
        out[k] = take_mine ? mine[i++] : theirs[j++];
    }
}

/* merge_take_high -- :83-103: the highest `take`, filled from the back; ties
 * prefer theirs (mine is taken only when strictly greater). */
static void orc_take_high(const int64_t* mine, uint64_t nm, const int64_t* theirs,
                          uint64_t nt, uint64_t take, int64_t* out) {
    uint64_t i = nm, j = nt;
    for (uint64_t k = take; k-- > 0;) {
        int take_mine;
        if (i == 0) take_mine = 0;
        else if (j == 0) take_mine = 1;
        else take_mine = mine[i - 1] > theirs[j - 1];
        out[k] = take_mine ? mine[--i] : theirs[--j];
    }
}

/* merge_split -- :107-113 (keep: 0 = low, 1 = high). out has |mine| slots. */
void orc_merge_split(const int64_t* mine, uint64_t nm, const int64_t* theirs,
                     uint64_t nt, int keep_high, int64_t* out) {
    if (keep_high) orc_take_high(mine, nm, theirs, nt, nm, out);
    else orc_take_low(mine, nm, theirs, nt, nm, out);
}

/* merge_split_padded -- :115-134. Blocks are (reals, virtuals); virtual
 * sentinels order above every real. Writes the kept reals to out_reals and
 * returns the kept virtual count through out_virtuals; *out_nreals gets the
 * real count. */
void orc_merge_split_padded(const int64_t* mine, uint64_t nm, uint64_t mine_virt,
                            const int64_t* theirs, uint64_t nt, uint64_t theirs_virt,
                            int keep_high, int64_t* out_reals, uint64_t* out_nreals,
                            uint64_t* out_virtuals) {
    const uint64_t width = nm + mine_virt;
    const uint64_t total_reals = nm + nt;
    if (!keep_high) {
        const uint64_t take = width < total_reals ? width : total_reals;
        orc_take_low(mine, nm, theirs, nt, take, out_reals);
        *out_nreals = take;
        *out_virtuals = width - take;
    } else {
        const uint64_t total_virt = mine_virt + theirs_virt;
        const uint64_t virt = width < total_virt ? width : total_virt;
        orc_take_high(mine, nm, theirs, nt, width - virt, out_reals);
        *out_nreals = width - virt;
        *out_virtuals = virt;
    }
}

/* parallel::scatter_merge_sort -- P/src/parallel_sort.cpp:166-254, restated as
 * a sequential simulation of the p rank programs. The result is the same
 * array the threaded reference gathers at the master:
 *   scatter by plan_partition (:186-193), local merge_sort (:200-215),
 *   p odd-even phases of merge_split_padded at width ceil(n/p) (:217-244),
 *   rank-order gather (:246-248).
 * Returns 0, -1 for p < 1, -2 on allocation failure. */
int orc_scatter_merge_sort(const int64_t* data, uint64_t n, int p, int64_t* out) {
    if (p < 1) return -1;
    uint64_t* sizes = (uint64_t*)malloc((size_t)p * sizeof(uint64_t));
    if (!sizes) return -2;
    orc_plan_partition(n, p, sizes);
    const uint64_t width = sizes[0];
    /* per-rank block storage: reals + count */
    int64_t** blk = (int64_t**)calloc((size_t)p, sizeof(int64_t*));
    int64_t** nxt = (int64_t**)calloc((size_t)p, sizeof(int64_t*));
    uint64_t* nreal = (uint64_t*)malloc((size_t)p * sizeof(uint64_t));
    uint64_t* nnext = (uint64_t*)malloc((size_t)p * sizeof(uint64_t));
    int64_t* scratch = (int64_t*)malloc((width ? width : 1) * sizeof(int64_t));
    int* partners = (int*)malloc((size_t)p * (size_t)p * sizeof(int));
    int rc = 0;
    if (!blk || !nxt || !nreal || !nnext || !scratch || !partners) { rc = -2; goto done; }
    {
        uint64_t off = 0;
        for (int r = 0; r < p; ++r) {
            blk[r] = (int64_t*)malloc((width ? width : 1) * sizeof(int64_t));
            nxt[r] = (int64_t*)malloc((width ? width : 1) * sizeof(int64_t));
            if (!blk[r] || !nxt[r]) { rc = -2; goto done; }
            memcpy(blk[r], data + off, sizes[r] * sizeof(int64_t));
            nreal[r] = sizes[r];
            off += sizes[r];
            orc_merge_sort_i64(blk[r], 0, (int64_t)nreal[r] - 1, scratch);
        }
    }
    orc_build_schedule(p, partners);
    for (int phase = 0; phase < p; ++phase) {
        const int* row = partners + (size_t)phase * (size_t)p;
        for (int r = 0; r < p; ++r) {
            const int q = row[r];
            if (q < 0) { nnext[r] = (uint64_t)-1; continue; }
            uint64_t virt_out = 0;
            orc_merge_split_padded(blk[r], nreal[r], width - nreal[r], blk[q], nreal[q],
                                   width - nreal[q], r < q ? 0 : 1, nxt[r], &nnext[r],
                                   &virt_out);
        }
        for (int r = 0; r < p; ++r) {
            if (nnext[r] == (uint64_t)-1) continue;
            int64_t* t = blk[r];
            blk[r] = nxt[r];
            nxt[r] = t;
            nreal[r] = nnext[r];
        }
    }
    {
        uint64_t off = 0;
        for (int r = 0; r < p; ++r) {
            memcpy(out + off, blk[r], nreal[r] * sizeof(int64_t));
            off += nreal[r];
        }
    }
done:
    if (blk) for (int r = 0; r < p; ++r) free(blk[r]);
    if (nxt) for (int r = 0; r < p; ++r) free(nxt[r]);
    free(blk); free(nxt); free(nreal); free(nnext); free(scratch); free(partners); free(sizes);
    return rc;
}

/* bench::verify_output / kernels::is_sorted -- P/src/bench.cpp:95-104,
 * P/src/sort_core.cpp:146-151. */
int orc_is_sorted_i64(const int64_t* s, uint64_t n) {
    for (uint64_t i = 1; i < n; ++i) if (s[i - 1] > s[i]) return 0;
    return 1;
}

/* Order-sensitive 64-bit fingerprint of a word sequence, used by the golden
 * fixtures: sum_i mix(x_i ^ mix(i + 1)) mod 2^64. Matches
 * oracle.fingerprint() in numpy. */
uint64_t orc_fingerprint_u64(const uint64_t* x, uint64_t n) {
    uint64_t h = 0;
    for (uint64_t i = 0; i < n; ++i) h += orc_mix(x[i] ^ orc_mix(i + 1));
    return h;
}
