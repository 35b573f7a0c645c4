// multi.cu -- the multi-GPU sample sort behind the C ABI (b2s_create_multi,
// b2s_sample_sort): one process, one host thread per GPU.
//
// Replaces parallel::scatter_merge_sort's distribution (P/src/parallel_sort.cpp:
// 166-254): the reference spawns p rank threads in one process
// (runtime::spawn_world, P/src/runtime.cpp:666-694) that scatter blocks from
// the master (:188-193), sort them (:200-215), run p odd-even merge-split
// phases of full-block send/recv (:217-244) and gather at the root
// (:246-248). Here rank r is a host thread driving GPU devices[r]:
//
//   (A) local onesweep radix sort of its shard, 64 regular samples
//   (B) all-gather of the samples (peer copies, or ncclAllGather), splitters
//       (identical on every rank), bucket bounds of the sorted shard
//   (C) all-gather of the bounds; the receive counts come to the host (one
//       small copy per rank: the merge and NCCL take host sizes)
//   (D) exchange + merge. p2p: the k-way merge kernels on GPU r read their
//       bucket's slice of every peer's sorted shard straight over NVLink
//       (cudaDeviceEnablePeerAccess), so the transfer rides the merge's loads
//       and no receive buffer exists. nccl: grouped ncclSend/ncclRecv
//       all-to-all into a receive buffer, then the k-way merge.
//
// Ordering between ranks is by CUDA events (a stream waits for a peer's
// event), never by a kernel spinning on another rank's flag, so emulated
// ranks (several ranks on one device) are safe on one GPU. Host threads meet
// at a barrier between the steps only so that every event a step waits on
// has been recorded. Output: bucket r on devices[r]; concatenated in rank
// order the buckets are the sorted array (the reference's gathered result),
// stable by global index (compound sample keys, ties to the lower rank).
//
// NCCL is loaded at run time (dlopen), so the library loads without it; the
// communicator is built with ncclCommInitAll over the distinct devices
// (NCCL refuses one device twice) and its asynchronous errors are polled
// while a step waits (B2S_ENCCL).
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "b2s_internal.cuh"

namespace b2s {
namespace {

// ---- NCCL, resolved at run time ------------------------------------------------
struct Nccl {
    bool ok = false;
    std::string why;
    int version = 0;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // the process may already hold an NCCL (torch's); dlopen returns it
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        bool all = true;
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            all = all && fp != nullptr;
        };
        sym(n.GetVersion, "ncclGetVersion");
        sym(n.GetErrorString, "ncclGetErrorString");
        sym(n.CommInitAll, "ncclCommInitAll");
        sym(n.CommDestroy, "ncclCommDestroy");
        sym(n.CommAbort, "ncclCommAbort");
        sym(n.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(n.AllGather, "ncclAllGather");
        sym(n.Send, "ncclSend");
        sym(n.Recv, "ncclRecv");
        sym(n.GroupStart, "ncclGroupStart");
        sym(n.GroupEnd, "ncclGroupEnd");
        if (!all) {
            n.why = "libnccl.so.2 lacks a required symbol";
            return;
        }
        n.GetVersion(&n.version);
        n.ok = true;
    });
    return n;
}

#define B2S_NCCL(call)                                                                        \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return ::b2s::set_error(B2S_ENCCL, "%s:%d %s -> %s", __FILE__, __LINE__, #call,    \
                                    nccl().GetErrorString(r_));                               \
    } while (0)

// ---- host barrier between the steps (threads of one call) --------------------
class Barrier {
   public:
    explicit Barrier(int n) : n_(n) {}
    void wait() {
        std::unique_lock<std::mutex> lk(m_);
        const unsigned long long gen = gen_;
        if (++count_ == n_) {
            count_ = 0;
            ++gen_;
            cv_.notify_all();
        } else {
            cv_.wait(lk, [&] { return gen_ != gen; });
        }
    }

   private:
    std::mutex m_;
    std::condition_variable cv_;
    int n_, count_ = 0;
    unsigned long long gen_ = 0;
};

}  // namespace
}  // namespace b2s

using namespace b2s;

struct b2s_multi {
    int G = 0;
    std::vector<int> dev;
    std::vector<b2s_ctx*> ctx;
    // per rank, on the rank's device
    std::vector<DevBuf> samples, all_samples, splitters, bounds, all_bounds;
    std::vector<DevBuf> sorted_k, sorted_v, recv_k, recv_v;
    std::vector<HostBuf> hbounds;
    std::vector<cudaEvent_t> ev_sorted, ev_bounds, ev_t[4];
    // transport
    bool peer_ok = true;  // every pair of distinct devices has peer access
    std::string peer_why;
    std::vector<ncclComm_t> comms;  // one per rank, when the devices are distinct
    std::string nccl_why;
    int transport = B2S_XCHG_AUTO;
    b2s_multi_timing last{};
    std::mutex call_m;  // one sample sort at a time per multi context
};

namespace {

bool nccl_usable(const b2s_multi* m) { return !m->comms.empty(); }

int pick_transport(const b2s_multi* m) {
    if (m->transport == B2S_XCHG_P2P) return m->peer_ok ? B2S_XCHG_P2P : -1;
    if (m->transport == B2S_XCHG_NCCL) return nccl_usable(m) ? B2S_XCHG_NCCL : -1;
    if (m->peer_ok) return B2S_XCHG_P2P;
    return nccl_usable(m) ? B2S_XCHG_NCCL : -1;
}

// Waits for a rank's stream, polling its NCCL communicator's asynchronous
// error (a failed or hung peer surfaces as B2S_ENCCL instead of a hang).
b2s_status wait_stream(b2s_multi* m, int r) {
    cudaStream_t s = m->ctx[r]->stream;
    if (m->comms.empty()) {
        B2S_CUDA(cudaStreamSynchronize(s));
        return B2S_OK;
    }
    for (;;) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return B2S_OK;
        if (e != cudaErrorNotReady) B2S_CUDA(e);
        ncclResult_t ae = ncclSuccess;
        B2S_NCCL(nccl().CommGetAsyncError(m->comms[r], &ae));
        if (ae != ncclSuccess && ae != ncclInProgress) {
            nccl().CommAbort(m->comms[r]);
            return set_error(B2S_ENCCL, "rank %d: NCCL asynchronous error: %s", r,
                             nccl().GetErrorString(ae));
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

struct Call {
    b2s_dtype dtype;
    const void* const* shards;
    const uint32_t* const* shard_vals;
    const uint64_t* counts;
    void* const* out;
    uint32_t* const* out_vals;
    const uint64_t* capacity;
    uint64_t* out_counts;
    int s;
    uint32_t flags;
    int transport;
};

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return 0.f;
    }
    return ms;
}

// One rank's part of the sample sort. Every step is attempted only while no
// rank has failed; every barrier is always reached, so a failing rank never
// strands the others.
void rank_main(b2s_multi* m, const Call& c, int r, Barrier& bar, std::vector<b2s_status>& st,
               std::vector<std::string>& msg, std::atomic<bool>& failed) {
    const int G = m->G;
    const size_t kb = (size_t)key_bytes(c.dtype);
    const bool vals = c.shard_vals != nullptr;
    const bool host = (c.flags & B2S_HOST) != 0;
    b2s_ctx* ctx = m->ctx[r];
    const uint64_t n = c.counts[r];
    uint64_t total = 0;
    std::vector<uint64_t> lens(G), offs(G);
    auto step = [&](auto&& fn) {
        if (failed.load()) return;
        const b2s_status s = fn();
        if (s != B2S_OK) {
            st[r] = s;
            msg[r] = b2s_last_error();
            failed.store(true);
        }
    };
    auto cuda = [&](cudaError_t e, const char* what) -> b2s_status {
        if (e == cudaSuccess) return B2S_OK;
        return set_error(e == cudaErrorMemoryAllocation ? B2S_ENOMEM : B2S_ECUDA, "rank %d: %s: %s", r, what,
                         cudaGetErrorString(e));
    };
    const bool timed = r == 0;
    // (A) local sort into the rank's exchange source, regular samples
    step([&]() -> b2s_status {
        B2S_TRY(cuda(cudaSetDevice(m->dev[r]), "cudaSetDevice"));
        if (timed) B2S_TRY(cuda(cudaEventRecord(m->ev_t[0][0], ctx->stream), "event"));
        B2S_TRY(m->sorted_k[r].ensure(std::max<uint64_t>(n, 1) * kb));
        if (vals) B2S_TRY(m->sorted_v[r].ensure(std::max<uint64_t>(n, 1) * 4));
        B2S_TRY(m->samples[r].ensure((size_t)c.s * sizeof(b2s_sample)));
        B2S_TRY(m->all_samples[r].ensure((size_t)c.s * G * sizeof(b2s_sample)));
        B2S_TRY(m->splitters[r].ensure((size_t)std::max(G - 1, 1) * sizeof(b2s_sample)));
        B2S_TRY(m->bounds[r].ensure((size_t)(G + 1) * 8));
        B2S_TRY(m->all_bounds[r].ensure((size_t)G * (G + 1) * 8));
        B2S_TRY(m->hbounds[r].ensure((size_t)G * (G + 1) * 8));
        const void* kin = c.shards[r];
        const uint32_t* vin = vals ? c.shard_vals[r] : nullptr;
        if (host && n > 0) {
            B2S_TRY(ctx->stage_in.ensure(n * kb));
            B2S_TRY(cuda(cudaMemcpyAsync(ctx->stage_in.ptr, kin, n * kb, cudaMemcpyHostToDevice, ctx->stream),
                         "shard upload"));
            kin = ctx->stage_in.ptr;
            if (vals) {
                B2S_TRY(ctx->stage_vin.ensure(n * 4));
                B2S_TRY(cuda(cudaMemcpyAsync(ctx->stage_vin.ptr, vin, n * 4, cudaMemcpyHostToDevice, ctx->stream),
                             "payload upload"));
                vin = static_cast<const uint32_t*>(ctx->stage_vin.ptr);
            }
        }
        if (n > 0)
            B2S_TRY(radix_sort(ctx, c.dtype, kin, m->sorted_k[r].ptr, vin,
                               vals ? static_cast<uint32_t*>(m->sorted_v[r].ptr) : nullptr, n));
        B2S_TRY(sample_regular(ctx, c.dtype, m->sorted_k[r].ptr, n, r, c.s,
                               static_cast<b2s_sample*>(m->samples[r].ptr)));
        if (timed) B2S_TRY(cuda(cudaEventRecord(m->ev_t[1][0], ctx->stream), "event"));
        return cuda(cudaEventRecord(m->ev_sorted[r], ctx->stream), "event");
    });
    bar.wait();
    // (B) all-gather of the samples, splitters, bucket bounds
    step([&]() -> b2s_status {
        b2s_sample* all = static_cast<b2s_sample*>(m->all_samples[r].ptr);
        const size_t sb = (size_t)c.s * sizeof(b2s_sample);
        if (c.transport == B2S_XCHG_NCCL) {
            B2S_NCCL(nccl().AllGather(m->samples[r].ptr, all, sb, ncclUint8, m->comms[r], ctx->stream));
        } else {
            for (int q = 0; q < G; ++q) {
                B2S_TRY(cuda(cudaStreamWaitEvent(ctx->stream, m->ev_sorted[q], 0), "wait"));
                B2S_TRY(cuda(cudaMemcpyPeerAsync(all + (size_t)q * c.s, m->dev[r], m->samples[q].ptr, m->dev[q], sb,
                                                 ctx->stream),
                             "sample copy"));
            }
        }
        b2s_sample* spl = static_cast<b2s_sample*>(m->splitters[r].ptr);
        B2S_TRY(select_splitters(ctx, all, c.s * G, G, spl));
        B2S_TRY(bucket_bounds(ctx, c.dtype, m->sorted_k[r].ptr, n, r, spl, G,
                              static_cast<uint64_t*>(m->bounds[r].ptr)));
        if (timed) B2S_TRY(cuda(cudaEventRecord(m->ev_t[2][0], ctx->stream), "event"));
        return cuda(cudaEventRecord(m->ev_bounds[r], ctx->stream), "event");
    });
    bar.wait();
    // (C) every rank's bounds; this rank's receive sizes to the host
    step([&]() -> b2s_status {
        uint64_t* ab = static_cast<uint64_t*>(m->all_bounds[r].ptr);
        const size_t bb = (size_t)(G + 1) * 8;
        if (c.transport == B2S_XCHG_NCCL) {
            B2S_NCCL(nccl().AllGather(m->bounds[r].ptr, ab, bb, ncclUint8, m->comms[r], ctx->stream));
        } else {
            for (int q = 0; q < G; ++q) {
                B2S_TRY(cuda(cudaStreamWaitEvent(ctx->stream, m->ev_bounds[q], 0), "wait"));
                B2S_TRY(cuda(cudaMemcpyPeerAsync(ab + (size_t)q * (G + 1), m->dev[r], m->bounds[q].ptr, m->dev[q], bb,
                                                 ctx->stream),
                             "bounds copy"));
            }
        }
        B2S_TRY(cuda(cudaMemcpyAsync(m->hbounds[r].ptr, ab, (size_t)G * bb, cudaMemcpyDeviceToHost, ctx->stream),
                     "bounds download"));
        B2S_TRY(wait_stream(m, r));
        const uint64_t* hb = static_cast<const uint64_t*>(m->hbounds[r].ptr);
        for (int q = 0; q < G; ++q) {
            lens[q] = hb[(size_t)q * (G + 1) + r + 1] - hb[(size_t)q * (G + 1) + r];
            offs[q] = total;
            total += lens[q];
        }
        c.out_counts[r] = total;
        if (total > c.capacity[r])
            return set_error(B2S_EINVAL, "rank %d: bucket of %llu keys exceeds out_capacity %llu", r,
                             (unsigned long long)total, (unsigned long long)c.capacity[r]);
        return B2S_OK;
    });
    bar.wait();
    // (D) exchange + k-way merge of the G runs of this bucket (ties to the lower
    // source rank: stable by global index)
    step([&]() -> b2s_status {
        const uint64_t* hb = static_cast<const uint64_t*>(m->hbounds[r].ptr);
        void* dout = c.out[r];
        uint32_t* dvout = vals ? c.out_vals[r] : nullptr;
        if (host) {
            B2S_TRY(ctx->stage_out.ensure(std::max<uint64_t>(total, 1) * kb));
            dout = ctx->stage_out.ptr;
            if (vals) {
                B2S_TRY(ctx->stage_vout.ensure(std::max<uint64_t>(total, 1) * 4));
                dvout = static_cast<uint32_t*>(ctx->stage_vout.ptr);
            }
        }
        B2S_TRY(ctx->alt_keys.ensure(std::max<uint64_t>(total, 1) * kb));
        if (vals) B2S_TRY(ctx->alt_vals.ensure(std::max<uint64_t>(total, 1) * 4));
        std::vector<const void*> runs(G);
        std::vector<const uint32_t*> vruns(G, nullptr);
        if (c.transport == B2S_XCHG_NCCL) {
            B2S_TRY(m->recv_k[r].ensure(std::max<uint64_t>(total, 1) * kb));
            if (vals) B2S_TRY(m->recv_v[r].ensure(std::max<uint64_t>(total, 1) * 4));
            char* rk = static_cast<char*>(m->recv_k[r].ptr);
            uint32_t* rv = static_cast<uint32_t*>(m->recv_v[r].ptr);
            const uint64_t* mine = hb + (size_t)r * (G + 1);  // this rank's bounds: what it sends
            const char* sk = static_cast<const char*>(m->sorted_k[r].ptr);
            const uint32_t* sv = static_cast<const uint32_t*>(m->sorted_v[r].ptr);
            B2S_NCCL(nccl().GroupStart());
            for (int q = 0; q < G; ++q) {
                const uint64_t sn = mine[q + 1] - mine[q];
                if (sn) B2S_NCCL(nccl().Send(sk + mine[q] * kb, sn * kb, ncclUint8, q, m->comms[r], ctx->stream));
                if (lens[q])
                    B2S_NCCL(nccl().Recv(rk + offs[q] * kb, lens[q] * kb, ncclUint8, q, m->comms[r], ctx->stream));
                if (vals) {
                    if (sn) B2S_NCCL(nccl().Send(sv + mine[q], sn * 4, ncclUint8, q, m->comms[r], ctx->stream));
                    if (lens[q]) B2S_NCCL(nccl().Recv(rv + offs[q], lens[q] * 4, ncclUint8, q, m->comms[r], ctx->stream));
                }
            }
            B2S_NCCL(nccl().GroupEnd());
            for (int q = 0; q < G; ++q) {
                runs[q] = rk + offs[q] * kb;
                if (vals) vruns[q] = rv + offs[q];
            }
        } else {
            // pull: the merge reads the peers' sorted shards in place (their
            // sorts finished before their bounds event, which this stream
            // waited for in step C)
            for (int q = 0; q < G; ++q) {
                const uint64_t lo = hb[(size_t)q * (G + 1) + r];
                runs[q] = static_cast<const char*>(m->sorted_k[q].ptr) + lo * kb;
                if (vals) vruns[q] = static_cast<const uint32_t*>(m->sorted_v[q].ptr) + lo;
            }
        }
        if (total > 0)
            B2S_TRY(kway_merge(ctx, c.dtype, runs.data(), vals ? vruns.data() : nullptr, lens.data(), G, dout, dvout,
                               ctx->alt_keys.ptr, static_cast<uint32_t*>(ctx->alt_vals.ptr)));
        if (timed) B2S_TRY(cuda(cudaEventRecord(m->ev_t[3][0], ctx->stream), "event"));
        if (host && total > 0) {
            B2S_TRY(cuda(cudaMemcpyAsync(c.out[r], dout, total * kb, cudaMemcpyDeviceToHost, ctx->stream),
                         "bucket download"));
            if (vals)
                B2S_TRY(cuda(cudaMemcpyAsync(c.out_vals[r], dvout, total * 4, cudaMemcpyDeviceToHost, ctx->stream),
                             "payload download"));
        }
        return wait_stream(m, r);
    });
    // the peers' pulls of this rank's shard are done once every rank passed
    // its own wait_stream: the caller joins all threads before returning
}

}  // namespace

extern "C" {

b2s_status b2s_create_multi(int ngpu, const int* devices, b2s_multi** out) {
    clear_error();
    if (out == nullptr) return set_error(B2S_EINVAL, "null output pointer");
    *out = nullptr;
    if (ngpu < 1 || devices == nullptr) return set_error(B2S_EINVAL, "need at least one device");
    if (ngpu > 64) return set_error(B2S_EINVAL, "at most 64 ranks");
    b2s_multi* m = new b2s_multi();
    m->G = ngpu;
    m->dev.assign(devices, devices + ngpu);
    auto fail = [&](b2s_status s) {
        const std::string e = b2s_last_error();
        b2s_destroy_multi(m);
        set_error(s, "%s", e.c_str());
        return s;
    };
    for (int r = 0; r < ngpu; ++r) {
        b2s_ctx* c = nullptr;
        const b2s_status s = b2s_create(devices[r], &c);
        if (s != B2S_OK) return fail(s);
        m->ctx.push_back(c);
    }
    m->samples.resize(ngpu);
    m->all_samples.resize(ngpu);
    m->splitters.resize(ngpu);
    m->bounds.resize(ngpu);
    m->all_bounds.resize(ngpu);
    m->sorted_k.resize(ngpu);
    m->sorted_v.resize(ngpu);
    m->recv_k.resize(ngpu);
    m->recv_v.resize(ngpu);
    m->hbounds.resize(ngpu);
    m->ev_sorted.resize(ngpu);
    m->ev_bounds.resize(ngpu);
    for (auto& v : m->ev_t) v.resize(1);
    for (int r = 0; r < ngpu; ++r) {
        cudaSetDevice(devices[r]);
        if (cudaEventCreateWithFlags(&m->ev_sorted[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&m->ev_bounds[r], cudaEventDisableTiming) != cudaSuccess)
            return fail(set_error(B2S_ECUDA, "cudaEventCreate failed"));
    }
    cudaSetDevice(devices[0]);
    for (auto& v : m->ev_t)
        if (cudaEventCreate(&v[0]) != cudaSuccess) return fail(set_error(B2S_ECUDA, "cudaEventCreate failed"));
    // peer access between every pair of distinct devices
    std::set<int> distinct(devices, devices + ngpu);
    for (int a : distinct) {
        for (int b : distinct) {
            if (a == b) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, a, b);
            if (!can) {
                m->peer_ok = false;
                m->peer_why = "no peer access from device " + std::to_string(a) + " to " + std::to_string(b);
                continue;
            }
            cudaSetDevice(a);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                m->peer_ok = false;
                m->peer_why = std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e);
            }
            cudaGetLastError();
        }
    }
    // NCCL communicator (one rank per device; NCCL rejects a device twice)
    if ((int)distinct.size() != ngpu) {
        m->nccl_why = "emulated ranks (a device appears more than once): NCCL needs distinct devices";
    } else if (!nccl().ok) {
        m->nccl_why = nccl().why;
    } else {
        m->comms.resize(ngpu);
        const ncclResult_t e = nccl().CommInitAll(m->comms.data(), ngpu, devices);
        if (e != ncclSuccess) {
            m->nccl_why = std::string("ncclCommInitAll: ") + nccl().GetErrorString(e);
            m->comms.clear();
        }
    }
    cudaSetDevice(devices[0]);
    *out = m;
    return B2S_OK;
}

b2s_status b2s_destroy_multi(b2s_multi* m) {
    if (m == nullptr) return B2S_OK;
    for (size_t r = 0; r < m->comms.size(); ++r)
        if (m->comms[r]) nccl().CommDestroy(m->comms[r]);
    for (int r = 0; r < (int)m->ctx.size(); ++r) {
        cudaSetDevice(m->dev[r]);
        cudaStreamSynchronize(m->ctx[r]->stream);
        for (auto* v : {&m->samples, &m->all_samples, &m->splitters, &m->bounds, &m->all_bounds, &m->sorted_k,
                        &m->sorted_v, &m->recv_k, &m->recv_v})
            if ((int)v->size() > r) (*v)[r].release();
        if ((int)m->hbounds.size() > r) m->hbounds[r].release();
        if ((int)m->ev_sorted.size() > r && m->ev_sorted[r]) cudaEventDestroy(m->ev_sorted[r]);
        if ((int)m->ev_bounds.size() > r && m->ev_bounds[r]) cudaEventDestroy(m->ev_bounds[r]);
    }
    if (!m->dev.empty()) cudaSetDevice(m->dev[0]);
    for (auto& v : m->ev_t)
        if (!v.empty() && v[0]) cudaEventDestroy(v[0]);
    for (b2s_ctx* c : m->ctx) b2s_destroy(c);
    delete m;
    return B2S_OK;
}

b2s_status b2s_multi_info(b2s_multi* m, int* ranks, int* p2p_ok, int* nccl_ok, int* nccl_version) {
    clear_error();
    if (m == nullptr) return set_error(B2S_EINVAL, "null multi context");
    if (ranks) *ranks = m->G;
    if (p2p_ok) *p2p_ok = m->peer_ok ? 1 : 0;
    if (nccl_ok) *nccl_ok = nccl_usable(m) ? 1 : 0;
    if (nccl_version) *nccl_version = nccl().ok ? nccl().version : 0;
    return B2S_OK;
}

b2s_status b2s_multi_set_transport(b2s_multi* m, int transport) {
    clear_error();
    if (m == nullptr) return set_error(B2S_EINVAL, "null multi context");
    if (transport < B2S_XCHG_AUTO || transport > B2S_XCHG_NCCL)
        return set_error(B2S_EINVAL, "unknown transport %d", transport);
    if (transport == B2S_XCHG_NCCL && !nccl_usable(m))
        return set_error(B2S_ENCCL, "NCCL transport unavailable: %s", m->nccl_why.c_str());
    if (transport == B2S_XCHG_P2P && !m->peer_ok)
        return set_error(B2S_EINVAL, "p2p transport unavailable: %s", m->peer_why.c_str());
    m->transport = transport;
    return B2S_OK;
}

b2s_status b2s_multi_get_timing(b2s_multi* m, b2s_multi_timing* out) {
    clear_error();
    if (m == nullptr || out == nullptr) return set_error(B2S_EINVAL, "null argument");
    *out = m->last;
    return B2S_OK;
}

b2s_status b2s_sample_sort(b2s_multi* m, b2s_dtype dtype, const void* const* shards,
                           const uint32_t* const* shard_vals, const uint64_t* counts, void* const* out,
                           uint32_t* const* out_vals, const uint64_t* out_capacity, uint64_t* out_counts,
                           int samples_per_gpu, uint32_t flags) {
    clear_error();
    if (m == nullptr) return set_error(B2S_EINVAL, "null multi context");
    if (!dtype_ok(dtype)) return set_error(B2S_EINVAL, "unknown dtype %d", (int)dtype);
    const int G = m->G;
    if (counts == nullptr || out_capacity == nullptr || out_counts == nullptr || shards == nullptr ||
        out == nullptr)
        return set_error(B2S_EINVAL, "null array argument");
    if ((shard_vals == nullptr) != (out_vals == nullptr))
        return set_error(B2S_EINVAL, "shard_vals and out_vals must both be set or both be NULL");
    if (samples_per_gpu < 1 || (long long)samples_per_gpu * G > 8192)
        return set_error(B2S_EINVAL, "samples_per_gpu * ranks must be in [1, 8192]");
    for (int r = 0; r < G; ++r) {
        if (counts[r] >= (1ull << 40)) return set_error(B2S_EINVAL, "shard %d too large", r);
        if (counts[r] > 0 && shards[r] == nullptr) return set_error(B2S_EINVAL, "shard %d is NULL", r);
        if (out_capacity[r] > 0 && out[r] == nullptr) return set_error(B2S_EINVAL, "out %d is NULL", r);
        if (shard_vals && counts[r] > 0 && shard_vals[r] == nullptr)
            return set_error(B2S_EINVAL, "shard_vals %d is NULL", r);
        if (out_vals && out_capacity[r] > 0 && out_vals[r] == nullptr)
            return set_error(B2S_EINVAL, "out_vals %d is NULL", r);
    }
    const int tr = pick_transport(m);
    if (tr < 0)
        return set_error(m->transport == B2S_XCHG_NCCL ? B2S_ENCCL : B2S_EINVAL,
                         "no exchange transport: p2p: %s; nccl: %s", m->peer_ok ? "ok" : m->peer_why.c_str(),
                         nccl_usable(m) ? "ok" : m->nccl_why.c_str());
    std::lock_guard<std::mutex> lk(m->call_m);
    Call c{dtype, shards, shard_vals, counts, out, out_vals, out_capacity, out_counts, samples_per_gpu, flags, tr};
    for (int r = 0; r < G; ++r) out_counts[r] = 0;
    Barrier bar(G);
    std::vector<b2s_status> st(G, B2S_OK);
    std::vector<std::string> msg(G);
    std::atomic<bool> failed{false};
    const auto t0 = std::chrono::steady_clock::now();
    // one host thread per rank, like runtime::spawn_world (P/src/runtime.cpp:683-688)
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r)
        th.emplace_back(rank_main, m, std::cref(c), r, std::ref(bar), std::ref(st), std::ref(msg), std::ref(failed));
    for (auto& t : th) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    cudaSetDevice(m->dev[0]);
    for (int r = 0; r < G; ++r)
        if (st[r] != B2S_OK) return set_error(st[r], "%s", msg[r].c_str());
    b2s_multi_timing t{};
    t.local_sort_ms = ev_ms(m->ev_t[0][0], m->ev_t[1][0]);
    t.splitters_ms = ev_ms(m->ev_t[1][0], m->ev_t[2][0]);
    t.exchange_merge_ms = ev_ms(m->ev_t[2][0], m->ev_t[3][0]);
    t.total_ms = std::chrono::duration<float, std::milli>(t1 - t0).count();
    t.transport = tr;
    t.max_bucket = 0;
    t.min_bucket = ~0ull;
    for (int r = 0; r < G; ++r) {
        t.max_bucket = std::max<uint64_t>(t.max_bucket, out_counts[r]);
        t.min_bucket = std::min<uint64_t>(t.min_bucket, out_counts[r]);
    }
    m->last = t;
    return B2S_OK;
}

}  // extern "C"
