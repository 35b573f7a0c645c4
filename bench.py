"""Benchmark: sorted keys/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload at every N: BASELINE.json configs[2] ("cfg3"), 2^31 int32 keys, the
gen_data splitmix64 stream (seed 1) >> 33, i.e. uniform over [0, 2^31), the
metric's "int32 at 1/2/4/8 B200" series. The total is fixed (strong scaling).

N=1: one GPU sorts all 2^31 keys (a pure local radix sort, 4 digit passes of
8 bits; the exchange of the sample sort is empty at G=1). One step = one
b2s_sort of the 8 GiB key array, input resident in HBM (larger than L2, so no
flush is needed). The line also carries cfg2's per-pass roofline (2^28 uint32,
BASELINE.json configs[1]) measured in the same run.

N>1 (torchrun, one process per GPU): the multi-GPU sample sort of the same
2^31 keys, shard r = plan_partition(2^31, N)[r] contiguous keys of the stream:
local sort, 64 regular samples per GPU, all-gather, splitters, bucket bounds,
exchange (merge kernels pull from peers over NVLink, or NCCL all-to-all), k-way
merge of the received runs.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libsortbench_ref.so, parallel::scatter_merge_sort, merge, p = k =
host threads) on the largest power-of-two sample of the workload that fits
the host's memory and the run's time budget (stated in the line).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted keys/sec"
UNIT = "keys/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic(_n, alg_bytes):
    """DRAM bytes per onesweep launch from the committed ncu --set full
    captures (profiles/r*_onesweep_traffic*.json, newest round first) of the
    launch with the same algorithmic bytes."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_onesweep_traffic*.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f))
            if d.get("algorithmic_bytes_per_launch") == alg_bytes:
                return d["traffic_bytes_per_launch"]
        except Exception:
            continue
    return None


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        """Starts sampling and waits (<= 5 s) for the first sample, so the
        sampler is live before the timed region begins."""
        try:
            fd, self.path = tempfile.mkstemp(prefix="clocks", suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 5 and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU arm (oracle/_ref = the reference library compiled from source)

N_TOTAL = 1 << 31
WORKLOAD = ("cfg3: 2^31 int32 keys (gen_data >> 33), sharded over the GPUs by plan_partition; "
            "G=1: one local radix sort (4 x 8-bit LSD passes), G>1: sample sort with 64 "
            "samples/GPU")
REF_BYTES_PER_KEY = 44  # peak RSS of scatter_merge_sort: 5.4 int64 copies


def _mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 16 << 30


def _ref_keys(n: int, shift: int = 33):
    """The workload's keys widened to int64 (the reference's only Element type)."""
    import numpy as np

    import oracle
    z = oracle.gen_data(n, 1).view(np.uint64)
    return (z >> np.uint64(shift)).astype(np.int64)


def ref_sample_size(budget_s: float, cap: int = N_TOTAL) -> tuple[int, str]:
    """Largest power of two <= cap whose reference run fits in half the host's
    available memory (44 B/key) and, extrapolated n log n from a 2^22 probe,
    in budget_s seconds."""
    import oracle
    threads = max(1, min(os.cpu_count() or 1, 64))
    if not oracle.ref_available():
        return 1 << 22, "oracle port (reference library not built)"
    probe = 1 << 22
    _, t = oracle.ref_scatter_merge_sort(_ref_keys(probe), threads, "merge", cores=threads, wall=True)
    mem = _mem_available() // 2
    n = probe
    while n * 2 <= cap:
        m = n * 2
        est = t * (m / probe) * ((m.bit_length() - 1) / 22)
        if est > budget_s or m * REF_BYTES_PER_KEY > mem:
            break
        n = m
    why = (f"largest power of two within half the host's available memory ({mem >> 30} GiB at "
           f"{REF_BYTES_PER_KEY} B/key) and ~{budget_s:.0f} s per run (2^22 probe: {t:.3f} s)")
    return n, why


def cpu_reference(sample_n: int, reps: int = 3, shift: int = 33, data=None):
    """parallel::scatter_merge_sort (merge, wall mode, p = k = host threads) on
    `sample_n` keys of the workload's distribution widened to int64;
    run_benchmark's semantics: median of reps of the world's wall seconds
    (P/src/bench.cpp:106-169)."""
    import oracle
    threads = max(1, min(os.cpu_count() or 1, 64))
    if data is None:
        data = _ref_keys(sample_n, shift)
    if oracle.ref_available():
        kind = "reference"
        times = []
        for _ in range(reps):
            out, secs = oracle.ref_scatter_merge_sort(data, threads, "merge", cores=threads,
                                                      wall=True)
            times.append(secs)
        t = sorted(times)[(len(times) - 1) // 2]
    else:  # the C restatement, single thread
        kind, threads = "port", 1
        t0 = time.perf_counter()
        out = oracle.scatter_merge_sort(data, 1)
        t = time.perf_counter() - t0
    if not (out[1:] >= out[:-1]).all():
        raise RuntimeError("CPU baseline produced unsorted output")
    return {"value": sample_n / t, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{sample_n} keys (gen_data >> {shift}, widened to int64), "
                      f"scatter_merge_sort merge p=k={threads}, median of {reps} wall-mode reps"}


def run_reference_arm(args, rank: int, world: int):
    if rank != 0:
        return
    # every step is one reference run; the whole --steps/--warmup run stays
    # within ~4 minutes
    per_step = 240.0 / max(1, args.steps + args.warmup)
    sample_n, why = (args.ref_sample, "set by --ref-sample") if args.ref_sample else \
        ref_sample_size(per_step)
    vals = []
    base = None
    data = _ref_keys(sample_n)  # generated once; each step sorts a fresh copy inside the reference
    for i in range(args.warmup + args.steps):
        b = cpu_reference(sample_n, reps=1, data=data)
        if i >= args.warmup:
            vals.append(b["value"])
        base = b
    v = statistics.median(vals)
    t_ms = sample_n / v * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (gen_data splitmix64 seed 1 >> 33)",
        "config": {"workload": WORKLOAD, "n": N_TOTAL, "sample_n": sample_n, "sample_why": why,
                   "p": base["cores"], "algorithm": "merge",
                   "note": "reference CPU path (host cores of the GPU box) on a bounded sample "
                           "of the workload"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": base["cores"], "kind": base["kind"],
                         "sample": base["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm, N = 1

def _pass_roofline(ctx, keys, out, reps, hbm_peak, peak_kind, kbytes, kernel):
    """Per-pass CUDA-event durations of the onesweep launches (events recorded
    inside the ABI on the launching stream) -> the roofline object."""
    ctx.enable_timing(True)
    pass_ms, hist_ms, executed = [], [], 0
    for _ in range(reps):
        ctx.sort(keys, out=out)
        t = ctx.timing()
        pass_ms.extend(t.pass_ms)
        hist_ms.append(t.hist_ms)
        executed = t.passes_executed
    ctx.enable_timing(False)
    n = keys.numel()
    avg_pass = statistics.mean(pass_ms)
    alg = 2 * kbytes * n  # read + write of every key per pass
    achieved = alg / (avg_pass * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "traffic": _traffic(n, alg),
            "kernel": kernel, "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": alg, "avg_launch_ms": avg_pass}
    phases = {"hist_plus_plan": statistics.mean(hist_ms), "pass_avg": avg_pass,
              "passes_executed": executed}
    return roof, phases


def _plan_partition(n: int, p: int):
    """plan_partition (P/src/parallel_sort.cpp:26-38): the first n mod p ranks
    get one extra key."""
    return [n // p + (1 if r < n % p else 0) for r in range(p)]


def run_single(args):
    import numpy as np
    import torch

    from paper_1105_6040_b200 import _lib
    from paper_1105_6040_b200.device import Context

    hbm_peak, peak_kind = _peaks()
    torch.cuda.set_device(0)
    ctx = Context(0)
    n = args.n
    keys = ctx.gen_keys(n, 1, torch.int32, shift=33)
    out = torch.empty_like(keys)
    torch.cuda.synchronize()

    # correctness gate on the benchmarked data (untimed, like verify_output):
    # sorted, a permutation of the input and, at the golden size, equal to the
    # CPU-computed expected output (tests/golden/fullsize.json)
    _, _, ms_in = ctx.check_sorted(keys)
    ctx.sort(keys, out=out)
    inv, fp, ms_out = ctx.check_sorted(out)
    if inv != 0 or ms_in != ms_out:
        raise RuntimeError("bench: sorted output failed verification")
    gold = _golden("cfg3")
    golden_ok = (fp == int(gold["fp"])) if gold and gold["n"] == n else None
    if golden_ok is False:
        raise RuntimeError("bench: sorted output differs from the golden fingerprint")

    for _ in range(args.warmup):
        ctx.sort(keys, out=out)
    torch.cuda.synchronize()

    # timed region: K sorts, CUDA events on the stream the kernels run on
    stream = torch.cuda.current_stream()
    clocks = Clocks(0)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches0 = _lib.lib().b2s_kernel_launches()
    e0.record(stream)
    for _ in range(args.steps):
        ctx.sort(keys, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = _lib.lib().b2s_kernel_launches() - launches0
    total_ms = e0.elapsed_time(e1)
    ms_step = total_ms / args.steps
    roof, phases = _pass_roofline(ctx, keys, out, args.steps, hbm_peak, peak_kind, 4,
                                  "onesweep_kernel (one digit pass of 2^31 int32 keys)")
    clk = clocks.stop()

    # cfg2's per-pass roofline (2^28 uint32, BASELINE.json configs[1]), same run
    k2 = ctx.gen_keys(1 << 28, 1, torch.uint32, shift=32)
    o2 = torch.empty_like(k2)
    for _ in range(3):
        ctx.sort(k2, out=o2)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        ctx.sort(k2, out=o2)
    t1.record(stream)
    torch.cuda.synchronize()
    roof2, phases2 = _pass_roofline(ctx, k2, o2, args.steps, hbm_peak, peak_kind, 4,
                                    "onesweep_kernel (one digit pass of 2^28 uint32 keys)")
    roof2["sort_ms"] = t0.elapsed_time(t1) / args.steps
    roof2["keys_per_s"] = (1 << 28) / (roof2["sort_ms"] * 1e-3)
    roof2["phases_ms"] = phases2
    del k2, o2

    # end to end through the C ABI with pinned HOST buffers (H2D + sort + D2H),
    # a stream of host batches through b2s_sort_batch: batch i+1 uploads while
    # batch i sorts and batch i-1 downloads (PCIe full duplex)
    h_in = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_in.copy_(keys.cpu())
    h_out = torch.empty(n, dtype=torch.int32, pin_memory=True)
    del out
    torch.cuda.empty_cache()
    hin_np = h_in.numpy()
    hout_np = h_out.numpy()
    # one batch per timed step (the stream's fill and drain amortise over the
    # run, as in a serving loop), at most 24 (~5 s of PCIe)
    e2e_steps = max(3, min(args.steps, 24))
    ctx.sort_batch([hin_np] * 3, outs=[hout_np] * 3)  # warm the three staging buffers
    t0 = time.perf_counter()
    ctx.sort_batch([hin_np] * e2e_steps, outs=[hout_np] * e2e_steps)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if not (hout_np[1:] >= hout_np[:-1]).all():
        raise RuntimeError("bench: e2e output unsorted")
    t0 = time.perf_counter()
    ctx.sort(hin_np, out=hout_np)  # one unpipelined call, for reference
    e2e_single_s = time.perf_counter() - t0

    value = n / (ms_step * 1e-3)
    cpu = None
    if not args.no_cpu:
        cpu_n, why = ref_sample_size(6.0)
        cpu = cpu_reference(cpu_n, reps=3)
        cpu["sample_why"] = why
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "i32",
        "data": "synthetic (gen_data splitmix64 seed 1 >> 33, int32 uniform in [0, 2^31))",
        "config": {"workload": WORKLOAD, "n": n, "p": 1, "key_bytes": 4,
                   "golden_fingerprint_match": golden_ok,
                   "l2": "inputs (8 GiB) larger than L2; no flush"},
        "roofline": roof,
        "phases_ms": phases,
        "roofline_cfg2": roof2,
        "e2e": {"value": n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 4 * n,
                "d2h_bytes_per_step": 4 * n, "ms_per_step": e2e_s * 1e3,
                "path": f"b2s_sort_batch(B2S_HOST) over {e2e_steps} pinned 8 GiB host batches "
                        "(upload/sort/download of consecutive batches overlapped)",
                "single_call_ms": e2e_single_s * 1e3},
        "gpu_launches": launches,
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    ctx.close()


def _golden(name):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "fullsize.json")) as f:
            for c in json.load(f)["configs"]:
                if c["config"] == name:
                    return c
    except Exception:
        pass
    return None


# ---------------------------------------------------------------------------
# B200 arm, N > 1 (torchrun)

def run_multi(args, rank: int, world: int):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1105_6040_b200 import _lib
    from paper_1105_6040_b200.device import Context
    from paper_1105_6040_b200.sample_sort import SampleSorter

    hbm_peak, peak_kind = _peaks()
    nvlink_gbs = 770.0  # measured peer copy per direction (B200_PROFILING.md)
    local = int(os.environ.get("LOCAL_RANK", rank))
    if rank == 0:  # NCCL's communicator-init lines (rank count) on rank 0's stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    print(f"[bench] rank {rank}/{world} on cuda:{local}: NCCL process group up", file=sys.stderr,
          flush=True)
    ctx = Context(local)
    total = args.n
    sizes = _plan_partition(total, world)
    n_local = sizes[rank]
    first = sum(sizes[:rank])
    # shard r = plan_partition's r-th contiguous slice of the cfg3 stream (int32 = z >> 33)
    keys = ctx.gen_keys(n_local, 1, torch.int32, shift=33, first=first)
    transport, transport_note = args.transport, None
    if transport == "p2p":
        probe = SampleSorter(ctx, transport="p2p")
        ok, err = probe.p2p_available()
        if not ok:  # every rank takes the same branch (collective probe)
            transport, transport_note = "nccl", f"p2p unavailable on this box: {err or 'a peer failed'}"
    sorter = SampleSorter(ctx, samples_per_rank=64, force_exchange=args.force_dist,
                          transport=transport)
    out, _ = sorter.sort(keys)
    if not sorter.verify(out, keys):
        raise RuntimeError(f"rank {rank}: sample sort verification failed")
    for _ in range(args.warmup):
        sorter.sort(keys)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.lib().b2s_kernel_launches()
    e0.record()
    for _ in range(args.steps):
        sorter.sort(keys)
    e1.record()
    torch.cuda.synchronize()
    launches = _lib.lib().b2s_kernel_launches() - launches0
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = float(ms.item())
    phases = dict(sorter.last_phase_ms)
    buckets = list(sorter.last_bucket_sizes)

    # per-pass kernel time of the local sort (CUDA events inside the ABI)
    ctx.enable_timing(True)
    pass_ms = []
    for _ in range(max(2, args.steps // 2)):
        ctx.sort(keys)
        pass_ms.extend(ctx.timing().pass_ms)
    ctx.enable_timing(False)
    clk = clocks.stop()

    # end to end through the public API: pinned host shard -> device -> sort ->
    # this rank's bucket back to pinned host memory, every step. The upload of
    # step i+1 (its own stream, its own device buffer) overlaps the sort of
    # step i, whose download runs on a third stream (PCIe is full duplex).
    h_in = torch.empty(n_local, dtype=torch.int32, pin_memory=True)
    h_in.copy_(keys.cpu())
    h_out = torch.empty(2 * n_local + 64 * world * world, dtype=torch.int32, pin_memory=True)
    comp = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    dbuf = [torch.empty_like(keys), torch.empty_like(keys)]
    ev_up = [torch.cuda.Event(), torch.cuda.Event()]
    ev_used = [None, None]  # the sort that read dbuf[b] last
    e2e_steps = max(2, min(args.steps, 24))
    dist.barrier()
    t0 = time.perf_counter()
    d2h = 0
    with torch.cuda.stream(up):
        dbuf[0].copy_(h_in, non_blocking=True)
        ev_up[0].record(up)
    for i in range(e2e_steps):
        b = i % 2
        comp.wait_event(ev_up[b])
        if i + 1 < e2e_steps:
            nb = (i + 1) % 2
            if ev_used[nb] is not None:
                up.wait_event(ev_used[nb])
            with torch.cuda.stream(up):
                dbuf[nb].copy_(h_in, non_blocking=True)
                ev_up[nb].record(up)
        ok_, _ = sorter.sort(dbuf[b])
        ev_used[b] = torch.cuda.Event()
        ev_used[b].record(comp)
        down.wait_event(ev_used[b])
        with torch.cuda.stream(down):
            h_out[: ok_.numel()].copy_(ok_, non_blocking=True)
        ok_.record_stream(down)  # the allocator must not hand it out before the download
        d2h = ok_.numel() * 4
    torch.cuda.synchronize()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device="cuda")
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)

    avg_pass = statistics.mean(pass_ms)
    alg = 2 * 4 * n_local
    achieved = alg / (avg_pass * 1e-3) / 1e9
    # combined roofline per GPU (serial, non-overlapped): the
    # prologue read, 4 sort passes and ONE merge pass over HBM, (G-1)/G of the
    # shard over NVLink each direction
    hbm_bytes = (4 * 2 * 4 + 4 + (2 * 4 if world > 1 else 0)) * n_local
    nvl_bytes = 4 * n_local * (world - 1) / world
    t_roof_ms = (hbm_bytes / (hbm_peak * 1e9) + nvl_bytes / (nvlink_gbs * 1e9)) * 1e3
    if rank == 0:
        line = {
            "metric": METRIC, "value": total / (ms_step * 1e-3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "i32",
            "data": "synthetic (gen_data splitmix64 seed 1 >> 33, int32 in [0, 2^31))",
            "config": {"workload": WORKLOAD, "n": total,
                       "n_per_gpu": n_local, "parallelism": f"sample sort over {world} GPUs",
                       "exchange": ("merge kernels pull buckets from peer shards over NVLink "
                                    "(CUDA IPC)" if transport == "p2p" else
                                    "NCCL all_to_all + k-way merge"),
                       "exchange_note": transport_note,
                       "l2": "inputs larger than L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": _traffic(n_local, alg),
                         "kernel": "onesweep_kernel (one digit pass, rank 0)",
                         "peak_kind": peak_kind,
                         "combined_hbm_nvlink_frac": t_roof_ms / ms_step,
                         "combined_roofline_ms": t_roof_ms,
                         "hbm_bytes_per_gpu": hbm_bytes,
                         "nvlink_bytes_per_gpu": nvl_bytes,
                         "nvlink_peak_gbs": nvlink_gbs,
                         "nvlink_peak_kind": "B200_PROFILING.md peer-copy figure (not measurable "
                                             "on the one-GPU development box)"},
            "phases_ms": phases, "bucket_sizes": buckets,
            "e2e": {"value": total / float(e2e_s.item()), "unit": UNIT,
                    "h2d_bytes_per_step": 4 * n_local, "d2h_bytes_per_step": d2h,
                    "path": "SampleSorter.sort from pinned host shards (per rank; upload of the "
                            "next step, sort and download overlapped on three streams)"},
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=N_TOTAL, help="total keys (all GPUs)")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="reference arm sample size (default: sized to memory and time)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="multi-GPU exchange: merge kernels pull from peers over NVLink "
                         "(CUDA IPC), or NCCL all-to-all + merge")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU sample-sort path even at world size 1")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1 or args.force_dist:
        run_multi(args, rank, world)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
