// b2s_internal.cuh -- shared definitions of the B200 sort kernels and host side.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "b200sort.h"

namespace b2s {

// ---------------------------------------------------------------------------
// error plumbing (thread-local message, status codes of b200sort.h)

b2s_status set_error(b2s_status st, const char* fmt, ...);
void clear_error();

#define B2S_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return ::b2s::set_error(e_ == cudaErrorMemoryAllocation ? B2S_ENOMEM        \
                                                                   : B2S_ECUDA,         \
                                    "%s:%d %s -> %s", __FILE__, __LINE__, #call,         \
                                    cudaGetErrorString(e_));                             \
    } while (0)

// One-time setup per device: kernel attributes (opt-in shared memory) are set
// per device, so a process driving several GPUs sets them on each. The setup
// runs under a mutex and the device counts as done only once it succeeded, so
// no thread launches before the attributes are set and a failure is retried.
struct DeviceOnce {
    std::mutex m;
    std::atomic<unsigned long long> done{0};
};
template <typename F>
b2s_status once_per_device(DeviceOnce& o, int device, F&& setup) {
    const unsigned long long bit = 1ull << (device & 63);
    if (o.done.load(std::memory_order_acquire) & bit) return B2S_OK;
    std::lock_guard<std::mutex> g(o.m);
    if (o.done.load(std::memory_order_relaxed) & bit) return B2S_OK;
    const b2s_status st = setup();
    if (st == B2S_OK) o.done.fetch_or(bit, std::memory_order_release);
    return st;
}

// every kernel launch of the library is counted (b2s_kernel_launches)
void note_launch();
unsigned long long launch_count();
void unnote_launches(unsigned long long n);  // launches recorded while capturing a graph
unsigned long long alloc_generation();       // bumped by every device scratch (re)allocation
#define B2S_LAUNCHED()                      \
    do {                                    \
        ::b2s::note_launch();               \
        B2S_CUDA(cudaGetLastError());       \
    } while (0)

#define B2S_TRY(expr)                                \
    do {                                             \
        b2s_status s_ = (expr);                      \
        if (s_ != B2S_OK) return s_;                 \
    } while (0)

// ---------------------------------------------------------------------------
// device scratch owned by a context, grown on demand, never shrunk

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    b2s_status ensure(size_t want);
    void release();
};

struct HostBuf {  // pinned
    void* ptr = nullptr;
    size_t bytes = 0;
    b2s_status ensure(size_t want);
    void release();
};

enum { kMaxSlots = 8 };

// Per-call radix sort plan, written on the device by radix_plan_kernel from
// the prologue's bit statistics so that constant-digit passes are skipped
// without a host round trip. Slot s runs digit position digit[s]; slots >=
// num_active exit at once.
struct RadixPlan {
    int num_active;
    int do_copy;        // 1: copy (in-place odd pass count / zero passes out of place), 2: reversed
    int need_fallback;  // first active digit is not digit 0: recount it
    int structured;     // input nearly sorted either way: swizzled staging
    int all_hist;       // every digit's histogram came from the prologue (no in-pass counting)
    int topfirst;       // 8-byte keys: only the upper four digits were sorted; the fix-up orders the ties
    int fix_flag;       // set by the fix-up when a tie run is too long for it: the full sort follows
    int digit[kMaxSlots];
    uint32_t dxor[kMaxSlots];  // 0x80 on the top digit of signed keys
    const unsigned long long* hist[kMaxSlots];  // digit histogram per slot
    const void* ksrc[kMaxSlots];
    void* kdst[kMaxSlots];
    const uint32_t* vsrc[kMaxSlots];
    uint32_t* vdst[kMaxSlots];
    const void* copy_ksrc;
    void* copy_kdst;
    const uint32_t* copy_vsrc;
    uint32_t* copy_vdst;
    unsigned int tile_counter[kMaxSlots];
};

// Device counters of one sort call, zeroed by one memset at the call's start.
struct RadixCounters {
    unsigned long long hist[kMaxSlots][256];  // slot s's digit histogram
    unsigned long long spec0[256];            // prologue's digit-0 histogram
    unsigned long long spec4[256];            // 8-byte keys, upper digits first: digit 4's histogram
    unsigned long long dhist[8][256];         // every digit's histogram (all-digit prologue)
    unsigned long long or_all;                // OR of all keys
    unsigned long long nor_all;               // OR of all complemented keys
    unsigned long long asc_pairs, desc_pairs;  // sampled adjacent pairs in order / reversed
    // every adjacent pair, counted by radix_order_check_kernel when the sample is all one way
    unsigned long long gt_pairs, lt_pairs, order_checked;
    unsigned long long ticket[256];            // keys-only first pass: digit offsets in tile arrival order
};

struct TimingEvents {
    cudaEvent_t ev[32];
    int used = 0;
};

}  // namespace b2s

struct b2s_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;

    // radix sort scratch
    b2s::DevBuf alt_keys, alt_vals;      // ping-pong partner / merge temp
    b2s::DevBuf seg_keys, seg_vals;      // partitioned sort: sorted segments
    b2s::DevBuf lookback;                // 2 regions x tiles x 256 words
    b2s::DevBuf hist;                    // 8 x 256 u64 (self-cleaning)
    b2s::DevBuf plan;                    // RadixPlan
    b2s::DevBuf parts;                   // merge-path partitions
    b2s::DevBuf misc;                    // small reductions
    b2s::HostBuf host_misc;              // pinned small results
    // B2S_HOST staging
    b2s::DevBuf stage_in, stage_out, stage_vin, stage_vout;
    // multi-GPU pull exchange: this rank's IPC-exported buffer (its sorted
    // shard) and the peers' buffers mapped into this process
    b2s::DevBuf xbuf;
    void* xbuf_handle_ptr = nullptr;  // allocation the cached handle belongs to
    unsigned char xbuf_handle[64] = {};
    std::vector<void*> xbuf_retired;  // outgrown exported buffers (peers may map them)
    std::map<std::string, void*> peers;  // IPC handle bytes -> mapped pointer
    // partitioned sort: per-partition scratch and side streams for the
    // concurrent local sorts
    b2s::DevBuf seg_lookback, seg_hist, seg_plan;
    b2s::DevBuf kmerge;  // grouped k-way merge: samples, tags, cuts
    b2s::DevBuf oe_keys;  // odd-even sort: two slots of width ceil(n/p) per block
    b2s::DevBuf zipf_table;  // b2s_gen_zipf's threshold table
    std::vector<cudaStream_t> side;
    std::vector<cudaEvent_t> side_done;
    cudaEvent_t fork = nullptr;
    // small partitioned sorts are bound by their chain of launches: the second
    // identical call (same buffers, sizes, p) is captured as a CUDA graph and
    // later ones replay it (b2s_partitioned_sort)
    cudaStream_t gstream = nullptr;
    cudaEvent_t g_in = nullptr, g_out = nullptr;
    cudaGraphExec_t gexec = nullptr;
    unsigned long long gkey[8] = {}, gseen[8] = {};
    bool gkey_valid = false, gseen_valid = false;
    unsigned long long glaunches = 0;  // kernels in the captured graph

    bool timing = false;
    cudaEvent_t ev[40] = {};
    int n_events = 0;
    b2s_timing last{};
    // event indices of the last call (-1 when absent)
    int ev_hist0 = -1, ev_hist1 = -1, ev_pass[b2s::kMaxSlots + 1] = {}, ev_copy1 = -1;
    int ev_merge0 = -1, ev_merge1 = -1;
    int last_passes_possible = 0;
    int last_merge_rounds = 0;
    bool have_sort = false, have_merge = false;
    // lane-ordered shared atomics verified on this device (onesweep ranks by
    // atomics instead of ballot matching); see b2s::probe_lane_order
    bool atomic_rank = false;
};

namespace b2s {

inline int key_bytes(b2s_dtype t) { return (t == B2S_I32 || t == B2S_U32) ? 4 : 8; }
inline bool key_signed(b2s_dtype t) { return t == B2S_I32 || t == B2S_I64; }
inline bool dtype_ok(int t) { return t >= B2S_I32 && t <= B2S_U64; }

// timing helpers (no-ops unless ctx->timing)
int record(b2s_ctx* ctx);
void timing_reset(b2s_ctx* ctx);

// The scratch one sort uses; by default the context's own buffers. Several
// sorts run concurrently (on different streams) each with its own set.
struct SortScratch {
    void* alt_keys;          // n keys: ping-pong partner
    uint32_t* alt_vals;      // n payload words (or null)
    void* lookback;          // 2 * lookback_region_bytes(n, ...) + 16
    RadixCounters* ctr;
    RadixPlan* plan;
};
size_t lookback_region_bytes(uint64_t n, int kbytes, bool vals);  // one region, for the tile actually launched
constexpr int kSideStreams = 8;  // concurrent partition sorts

// device entry points implemented in the .cu files (all async on ctx->stream)
b2s_status radix_sort(b2s_ctx* ctx, b2s_dtype dtype, const void* kin, void* kout,
                      const uint32_t* vin, uint32_t* vout, uint64_t n,
                      const SortScratch* scratch = nullptr);
b2s_status kway_merge(b2s_ctx* ctx, b2s_dtype dtype, const void* const* runs,
                      const uint32_t* const* vals, const uint64_t* lens, int k, void* out,
                      uint32_t* vout, void* tmp, uint32_t* vtmp);
b2s_status merge_split_padded(b2s_ctx* ctx, b2s_dtype dtype, const void* mine, uint64_t nm,
                              uint64_t mv, const void* theirs, uint64_t nt, uint64_t tv,
                              int keep_high, void* out, uint64_t* out_n, uint64_t* out_v);
b2s_status sample_regular(b2s_ctx* ctx, b2s_dtype dtype, const void* keys, uint64_t n,
                          int rank, int s, b2s_sample* out);
b2s_status select_splitters(b2s_ctx* ctx, const b2s_sample* samples, int count, int nparts,
                            b2s_sample* splitters);
b2s_status bucket_bounds(b2s_ctx* ctx, b2s_dtype dtype, const void* keys, uint64_t n, int rank,
                         const b2s_sample* splitters, int nparts, uint64_t* bounds);
b2s_status probe_lane_order(b2s_ctx* ctx, bool* ok);
b2s_status partitioned_sort_dev(b2s_ctx* ctx, b2s_dtype dtype, const void* din, void* dout,
                                const uint32_t* dvin, uint32_t* dvout, uint64_t n, int p);
b2s_status gen_keys(b2s_ctx* ctx, b2s_dtype dtype, uint64_t first, uint64_t n, uint64_t seed,
                    int shift, void* out);
b2s_status check_sorted(b2s_ctx* ctx, b2s_dtype dtype, const void* keys, uint64_t n,
                        uint64_t* inv, uint64_t* fp, uint64_t* ms);
b2s_status gen_zipf(b2s_ctx* ctx, b2s_dtype dtype, uint64_t first, uint64_t n, uint64_t seed,
                    const uint64_t* thresholds, uint32_t nvalues, void* out);

// ---------------------------------------------------------------------------
// device helpers

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

}  // namespace b2s
