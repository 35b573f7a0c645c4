/*
 * b200sort.h -- C ABI of the B200-native partitioned sort.
 *
 * This is the drop-in boundary for the hot path of the reference
 * (/root/reference/proj, "sortbench"): scatter N keys over p partitions, sort
 * each partition, merge the sorted runs into one ascending array. The
 * reference's C++ entry points keep their signatures in
 * include/sortbench_b200/ and call down into these
 * functions; nothing here uses C++ or torch types.
 *
 * Conventions
 *   - Every function returns a b2s_status; on failure b2s_last_error() (a
 *     thread-local string) says why. The reference throws instead
 *     (P/include/sortbench/errors.hpp:10-46); the shims map EINVAL ->
 *     ConfigError, EINTERNAL -> ProgrammingError, the rest -> runtime_error.
 *   - Pointers are DEVICE pointers unless the call takes `flags` and
 *     B2S_HOST is set, in which case they are host pointers (pinned memory
 *     gives full PCIe bandwidth) and the call is synchronous.
 *   - DEVICE calls are asynchronous on the context's stream (b2s_set_stream).
 *   - A context is bound to one device and must be used by one host thread
 *     at a time (the reference runs one rank per thread,
 *     P/src/runtime.cpp:683-688: give each thread its own context).
 *   - There is no CPU fallback: without a usable sm_100 device b2s_create
 *     fails with B2S_ECUDA.
 */
#ifndef B200SORT_H
#define B200SORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum b2s_status {
    B2S_OK = 0,
    B2S_EINVAL = 1,    /* bad argument / configuration   -> ConfigError      */
    B2S_ENOMEM = 2,    /* device or pinned allocation failed                 */
    B2S_ECUDA = 3,     /* CUDA runtime / launch error                        */
    B2S_EINTERNAL = 4, /* internal invariant violated    -> ProgrammingError */
    B2S_ENCCL = 5      /* NCCL error (init, collective, asynchronous abort) */
} b2s_status;

/* Key types. The reference sorts int64 only (Element,
 * P/include/sortbench/element.hpp:10); the GPU path also sorts the 32-bit and
 * unsigned widths named by BASELINE.json. Signed keys order as signed. */
typedef enum b2s_dtype { B2S_I32 = 0, B2S_U32 = 1, B2S_I64 = 2, B2S_U64 = 3 } b2s_dtype;

#define B2S_DEVICE 0u
#define B2S_HOST 1u

typedef struct b2s_ctx b2s_ctx;

/* Regular-sampling record used by the multi-GPU sample sort: `key` is the
 * key's order-preserving unsigned image (sign bit flipped for signed types),
 * `tag` = (rank << 40) | position-in-sorted-shard, so (key, tag) is a total
 * order that equals (key, global index) for a stable local sort. A slot with
 * key = tag = UINT64_MAX is empty. */
typedef struct b2s_sample {
    uint64_t key;
    uint64_t tag;
} b2s_sample;

/* Device-side phase timings of the most recent sort/merge call on a context
 * with timing enabled (CUDA events on the context's stream). */
typedef struct b2s_timing {
    float hist_ms;           /* upfront all-digit histogram + pass plan            */
    float pass_ms[8];        /* onesweep digit pass per executed slot               */
    int passes_executed;     /* digit passes that ran (constant digits are skipped) */
    int passes_possible;     /* 4 for 32-bit keys, 8 for 64-bit keys                */
    float copy_ms;           /* trailing copy (odd pass count in place), else 0     */
    float merge_ms;          /* merge-path rounds (b2s_merge / partitioned sort)    */
    int merge_rounds;
    float total_ms;          /* first event to last event of the call               */
} b2s_timing;

/* ---- context ----------------------------------------------------------- */
b2s_status b2s_create(int device, b2s_ctx** out);
b2s_status b2s_destroy(b2s_ctx* ctx);
/* `stream` is a cudaStream_t (NULL = the legacy default stream). A new
 * context starts on its own non-blocking stream. */
b2s_status b2s_set_stream(b2s_ctx* ctx, void* stream);
b2s_status b2s_synchronize(b2s_ctx* ctx);
b2s_status b2s_enable_timing(b2s_ctx* ctx, int on);
b2s_status b2s_get_timing(b2s_ctx* ctx, b2s_timing* out);
const char* b2s_last_error(void);
const char* b2s_version(void);
int b2s_device_count(void);
/* Kernels this library has launched in this process (all contexts); the
 * difference across a region counts the region's launches. */
unsigned long long b2s_kernel_launches(void);
/* 1 when the context ranks keys with lane-ordered shared atomics (the probe
 * at b2s_create found same-word lanes of one atomic served in lane order on
 * this device), 0 when it fell back to ballot matching (also B2S_RANK=ballot);
 * -1 for a bad context. Both are stable; the atomic ranking is the fast one. */
int b2s_lane_ordered_atomics(b2s_ctx* ctx);

/* ---- multi-GPU pull exchange (one process per GPU) ------------------------
 * Replaces the reference's rank-to-rank block messages (Comm::send/recv and
 * gather, P/src/runtime.cpp:219-328,547-568): every rank exports the buffer
 * holding its sorted shard, maps its peers' buffers, and its merge kernel
 * reads its bucket's slice of every peer's shard straight over NVLink.
 *
 * b2s_exchange_buffer: a device buffer of at least `bytes` owned by the
 *   context (reused across calls, reallocated when it must grow) and its CUDA
 *   IPC handle (64 bytes) for the peers.
 * b2s_open_peer: maps a peer's buffer from its handle (cached per handle;
 *   the same process may not open its own handle).
 * b2s_close_peers: unmaps every peer buffer this context opened. */
b2s_status b2s_exchange_buffer(b2s_ctx* ctx, uint64_t bytes, void** ptr, void* handle64);
b2s_status b2s_open_peer(b2s_ctx* ctx, const void* handle64, void** ptr);
b2s_status b2s_close_peers(b2s_ctx* ctx);

/* ---- local sort ----------------------------------------------------------
 * Replaces the per-rank comparison kernels behind KernelFn
 * (P/include/sortbench/parallel_sort.hpp:69-72; kernels::merge_sort /
 * quick_sort / bubble_sort, P/src/sort_core.cpp:23-144) with an LSD onesweep
 * radix sort. keys_in -> keys_out (they may alias: in-place). vals_in/vals_out
 * are an optional uint32 payload (both NULL or both non-NULL) permuted with
 * the keys; the sort is stable, so equal keys keep their payload order. */
b2s_status b2s_sort(b2s_ctx* ctx, b2s_dtype dtype, const void* keys_in, void* keys_out,
                    const uint32_t* vals_in, uint32_t* vals_out, uint64_t n, uint32_t flags);

/* Sorts `count` independent host arrays of n keys each (B2S_HOST only):
 * keys_in[i] -> keys_out[i] (and optional payloads). The host->device copy of
 * array i+1, the sort of array i and the device->host copy of array i-1 run
 * concurrently on three streams (PCIe is full duplex), so a stream of batches
 * is bounded by the slower copy direction, not by copy + sort + copy. Pinned
 * host memory is required for the overlap. Synchronous. */
b2s_status b2s_sort_batch(b2s_ctx* ctx, b2s_dtype dtype, const void* const* keys_in,
                          void* const* keys_out, const uint32_t* const* vals_in,
                          uint32_t* const* vals_out, uint64_t n, int count, uint32_t flags);

/* ---- k-way merge ---------------------------------------------------------
 * Replaces the odd-even merge_split phases + rank-order gather of the root
 * merge (P/src/parallel_sort.cpp:59-134,217-248): merges k sorted runs into
 * `out`, stably, ties taken from the lower run index (kernels::merge_runs'
 * rule, P/src/sort_core.cpp:46). `runs`, `run_vals` and `lens` are HOST
 * arrays of k entries; the run pointers are device pointers (or host pointers
 * with B2S_HOST). `out` must not overlap any run. */
b2s_status b2s_merge(b2s_ctx* ctx, b2s_dtype dtype, const void* const* runs,
                     const uint32_t* const* run_vals, const uint64_t* lens, int k, void* out,
                     uint32_t* out_vals, uint32_t flags);

/* ---- whole single-GPU path ----------------------------------------------
 * parallel::scatter_merge_sort on one device (P/src/parallel_sort.cpp:166-254):
 * split `in` into p contiguous partitions by plan_partition (:26-38), sort
 * each partition, merge the p runs into `out` (may alias `in`). p >= 1. */
b2s_status b2s_partitioned_sort(b2s_ctx* ctx, b2s_dtype dtype, const void* in, void* out,
                                const uint32_t* vals_in, uint32_t* vals_out, uint64_t n,
                                int p, uint32_t flags);

/* plan_partition (P/src/parallel_sort.cpp:26-38): the first n mod p
 * partitions get one extra key. sizes has p slots (host). */
b2s_status b2s_plan_partition(uint64_t n, int p, uint64_t* sizes);

/* The reference's own p-phase algorithm on one device, for comparison with
 * the merge of b2s_partitioned_sort: plan_partition scatter, a radix sort of
 * each block, p odd-even phases of merge_split_padded at width ceil(n/p)
 * between partner blocks (build_schedule, P/src/parallel_sort.cpp:40-55,
 * 217-244; every merge-split is a merge-path window on the device, the kept
 * counts follow from the widths on the host, so nothing synchronises), and
 * the rank-order gather into `out` (:246-248). Keys only, like the
 * reference. p >= 1. */
b2s_status b2s_odd_even_sort(b2s_ctx* ctx, b2s_dtype dtype, const void* in, void* out, uint64_t n,
                             int p, uint32_t flags);

/* ---- odd-even merge-split (the reference's own exchange step) -----------
 * merge_split_padded (P/src/parallel_sort.cpp:115-134) on the device: `mine`
 * and `theirs` are sorted runs padded with virtual top sentinels to the same
 * width; keeps the low (keep_high = 0) or high width elements. Writes the kept
 * reals to out_reals and their count / the kept virtual count to the host
 * integers. */
b2s_status b2s_merge_split_padded(b2s_ctx* ctx, b2s_dtype dtype, const void* mine,
                                  uint64_t n_mine, uint64_t mine_virtuals, const void* theirs,
                                  uint64_t n_theirs, uint64_t theirs_virtuals, int keep_high,
                                  void* out_reals, uint64_t* out_n_reals,
                                  uint64_t* out_virtuals, uint32_t flags);

/* ---- sample sort building blocks (one process per GPU) ------------------
 * These replace Comm::scatter/gather and the p odd-even phases
 * (P/src/runtime.cpp:509-568, P/src/parallel_sort.cpp:188-248) across GPUs:
 *   local b2s_sort -> b2s_sample_regular -> all-gather samples ->
 *   b2s_select_splitters -> b2s_bucket_bounds -> all-to-all -> b2s_merge.
 * All pointers are device pointers. */
b2s_status b2s_sample_regular(b2s_ctx* ctx, b2s_dtype dtype, const void* sorted_keys,
                              uint64_t n, int rank, int samples, b2s_sample* out);
b2s_status b2s_select_splitters(b2s_ctx* ctx, const b2s_sample* samples, int count,
                                int nparts, b2s_sample* splitters);
b2s_status b2s_bucket_bounds(b2s_ctx* ctx, b2s_dtype dtype, const void* sorted_keys,
                             uint64_t n, int rank, const b2s_sample* splitters, int nparts,
                             uint64_t* bounds);

/* ---- multi-GPU sample sort in one process --------------------------------
 * parallel::scatter_merge_sort across GPUs (P/src/parallel_sort.cpp:166-254):
 * the reference runs p rank threads in one process (runtime::spawn_world,
 * P/src/runtime.cpp:666-694) that scatter, sort, exchange blocks in p
 * odd-even phases of send/recv (:217-244) and gather at the root (:246-248).
 * Here one host thread per rank drives GPU devices[r]: local radix sort,
 * samples_per_gpu regular samples, all-gather, splitters, bucket bounds, ONE
 * exchange, and a k-way merge of the received runs.
 *
 * b2s_create_multi: one rank per entry of `devices`. A device may repeat
 *   (emulated ranks: each rank gets its own context and stream on it). Peer
 *   access is enabled between every pair of distinct devices; an NCCL
 *   communicator (ncclCommInitAll, NCCL loaded at run time) is built when the
 *   devices are distinct. Neither is an error when unavailable: the exchange
 *   transport is chosen per call.
 * Transport: B2S_XCHG_P2P -- the merge kernels of rank r read their bucket's
 *   slice of every peer's sorted shard over NVLink (no receive buffer);
 *   B2S_XCHG_NCCL -- grouped ncclSend/ncclRecv all-to-all, then the merge;
 *   B2S_XCHG_AUTO (default) -- p2p when every pair has peer access, else NCCL.
 * b2s_sample_sort (synchronous): shards[r] (counts[r] keys, device pointers on
 *   devices[r], or host pointers with B2S_HOST) -> bucket r in out[r]
 *   (capacity out_capacity[r] keys) with out_counts[r] keys. The buckets
 *   concatenated in rank order are the ascending array, stable by global
 *   index (shard order; ties to the lower rank), so payloads follow the
 *   reference's stable tie rule. A bucket above its capacity fails with
 *   B2S_EINVAL and out_counts holding the sizes needed. With 64 samples per
 *   GPU a bucket holds at most about 2 * total / ranks keys (regular
 *   sampling), also for all-equal keys (compound sample keys).
 *   samples_per_gpu * ranks <= 8192. */
#define B2S_XCHG_AUTO 0
#define B2S_XCHG_P2P 1
#define B2S_XCHG_NCCL 2
typedef struct b2s_multi b2s_multi;
typedef struct b2s_multi_timing {
    float local_sort_ms;      /* rank 0: local radix sort + regular samples          */
    float splitters_ms;       /* rank 0: sample all-gather, splitters, bucket bounds */
    float exchange_merge_ms;  /* rank 0: bounds, exchange and k-way merge            */
    float total_ms;           /* host wall time of the whole call                    */
    int transport;            /* B2S_XCHG_P2P or B2S_XCHG_NCCL                        */
    uint64_t max_bucket, min_bucket;
} b2s_multi_timing;
b2s_status b2s_create_multi(int ngpu, const int* devices, b2s_multi** out);
b2s_status b2s_destroy_multi(b2s_multi* m);
b2s_status b2s_multi_info(b2s_multi* m, int* ranks, int* p2p_ok, int* nccl_ok, int* nccl_version);
b2s_status b2s_multi_set_transport(b2s_multi* m, int transport);
b2s_status b2s_multi_get_timing(b2s_multi* m, b2s_multi_timing* out);
b2s_status b2s_sample_sort(b2s_multi* m, b2s_dtype dtype, const void* const* shards,
                           const uint32_t* const* shard_vals, const uint64_t* counts,
                           void* const* out, uint32_t* const* out_vals,
                           const uint64_t* out_capacity, uint64_t* out_counts,
                           int samples_per_gpu, uint32_t flags);

/* ---- input generation and verification ----------------------------------
 * b2s_gen_keys: key_i = (T)(z_{first+i} >> shift) where z is bench::gen_data's
 * splitmix64 stream for `seed` (P/src/bench.cpp:57-71) -- bit-identical to the
 * host generator. b2s_check_sorted: adjacent-inversion count, the golden
 * fixtures' order-sensitive fingerprint (sum_i mix(w_i ^ mix(i+1)) over the
 * int64/uint64 widening w) and an order-independent multiset hash
 * (sum_i mix(w_i)), all returned to host integers (synchronous). */
b2s_status b2s_gen_keys(b2s_ctx* ctx, b2s_dtype dtype, uint64_t first, uint64_t n,
                        uint64_t seed, int shift, void* out, uint32_t flags);
b2s_status b2s_check_sorted(b2s_ctx* ctx, b2s_dtype dtype, const void* keys, uint64_t n,
                            uint64_t* inversions, uint64_t* fingerprint, uint64_t* multiset,
                            uint32_t flags);
/* cfg4a's skewed input (BASELINE.json configs[3](a): Zipf s=1.2 over 2^20
 * values): key_i = the number of entries of the HOST table `thresholds`
 * (nvalues ascending uint64, last = 2^53) that are <= (z_{first+i} >> 11),
 * z = gen_data's stream for `seed`. Integer-only, so bit-identical to a host
 * draw from the same table (oracle.zipf_thresholds / oracle.zipf_keys). */
b2s_status b2s_gen_zipf(b2s_ctx* ctx, b2s_dtype dtype, uint64_t first, uint64_t n, uint64_t seed,
                        const uint64_t* thresholds, uint32_t nvalues, void* out, uint32_t flags);

#ifdef __cplusplus
}
#endif

#endif /* B200SORT_H */
