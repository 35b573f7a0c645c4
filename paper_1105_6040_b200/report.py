"""Benchmark reports and trace export in the reference's formats, for runs of
the partitioned sort on the GPU.

Mirrors sortbench's ``bench`` reporting layer (P/include/sortbench/bench.hpp,
P/src/bench.cpp): ``RunConfig`` / ``run_id`` (:30-50), ``run_benchmark``
(:106-169: median repetition, verification gate), ``overhead_ratio``
(:171-199), the experiment-1 CSV row and grid (:205-254) and the trace
JSONL + summary export (:335-395), byte-compatible with the reference's output
(``format_double`` follows std::to_chars' general format), so GPU and CPU runs
land in the same files and tables.

What a "rank" is on one GPU: the reference's p ranks each sort one block
(``compute``) and exchange blocks (``scatter``, odd-even ``send``/``recv``,
``gather``). Here rank r has its own context and CUDA stream (the reference's
one Comm per rank thread) and its ``compute`` event is the device time of the
radix sort of block r -- the ranks' sorts run concurrently -- and rank 0's
``gather`` event is the k-way merge of the p sorted blocks (the root merge);
scatter is free (blocks are views). Events are CUDA-event intervals in
nanoseconds from the run's first event, and ``wall_seconds`` spans the whole
run. Only wall mode exists on the GPU
(counted mode measures CPU operation counts); the operation counters a radix
sort cannot produce (comparisons, swaps, recursion depth) are 0.
``trace_from_sample_sort`` turns one multi-GPU SampleSorter run into the same
event kinds (compute / bcast / send / gather).
"""
from __future__ import annotations

import decimal
import json
import math
from dataclasses import dataclass, field

from .errors import ConfigError, VerificationError

ALGORITHMS = ("bubble", "merge", "quick")  # parallel::Algorithm order
EVENT_KINDS = ("compute", "send", "recv", "bcast", "scatter", "gather", "barrier", "idle")
EXP1_CSV_HEADER = "algorithm,n,m,k,time_s,weighted_ops,compute_s,overhead_s,ratio"


def format_double(v: float) -> str:
    """std::to_chars(general) of a double (P/src/bench.cpp:22-29): the
    shortest round-trip digits, scientific when the decimal exponent is < -4
    or >= 6, exponent with a sign and at least two digits."""
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    if v == 0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    sign, digits, exp = decimal.Decimal(repr(v)).as_tuple()
    ds = "".join(map(str, digits)).rstrip("0") or "0"
    # value = 0.d1d2... * 10^(x+1) with x the decimal exponent of d1
    x = exp + len(digits) - 1
    neg = "-" if sign else ""
    if x < -4 or x >= 6:
        mant = ds[0] + ("." + ds[1:] if len(ds) > 1 else "")
        return f"{neg}{mant}e{'-' if x < 0 else '+'}{abs(x):02d}"
    if x < 0:
        return f"{neg}0.{'0' * (-x - 1)}{ds}"
    if len(ds) <= x + 1:
        return neg + ds + "0" * (x + 1 - len(ds))
    return f"{neg}{ds[:x + 1]}.{ds[x + 1:]}"


@dataclass
class RunConfig:
    """bench::RunConfig (P/include/sortbench/bench.hpp:15-23)."""
    algorithm: str = "merge"
    n: int = 0
    procs: int = 1
    cores: int = 1
    seed: int = 1
    mode: str = "wall"
    repetitions: int = 1


def run_id(c: RunConfig) -> str:
    """FNV-1a 64 of "algorithm|n|procs|cores|seed|mode|repetitions", 16 hex
    digits (P/src/bench.cpp:30-50)."""
    key = f"{c.algorithm}|{c.n}|{c.procs}|{c.cores}|{c.seed}|{c.mode}|{c.repetitions}"
    h = 1469598103934665603
    for ch in key.encode():
        h ^= ch
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


@dataclass
class TraceEvent:
    """runtime::TraceEvent (P/include/sortbench/runtime.hpp:37-43)."""
    rank: int
    kind: str
    t_start: int
    t_end: int
    bytes: int = 0


@dataclass
class WorldReport:
    """The parts of runtime::WorldReport the exports read
    (P/include/sortbench/runtime.hpp:66-86)."""
    procs: int
    core_slots: int
    mode: str = "wall"
    wall_seconds: float = 0.0
    trace: list = field(default_factory=list)        # TraceEvent, ordered by (rank, time)
    counters: list = field(default_factory=list)     # per rank dict of the 7 counters
    weighted_ops: int = 0


@dataclass
class RunReport:
    """bench::RunReport (P/include/sortbench/bench.hpp:29-38)."""
    config: RunConfig
    wall_seconds: float
    weighted_ops: int
    compute_total: float
    overhead_total: float
    world: WorldReport


_COUNTERS = ("comparisons", "swaps", "element_moves", "messages_sent", "bytes_sent",
             "peak_tracked_elements", "max_recursion_depth")


def overhead_ratio(world: WorldReport) -> tuple[list, float]:
    """(per-rank overhead/compute, aggregate mean; inf when a rank has
    overhead but no compute) (P/src/bench.cpp:171-199)."""
    p = world.procs
    comp, over = [0.0] * p, [0.0] * p
    for ev in world.trace:
        (comp if ev.kind == "compute" else over)[ev.rank] += float(ev.t_end - ev.t_start)
    per, inf = [], False
    for r in range(p):
        if comp[r] > 0:
            per.append(over[r] / comp[r])
        elif over[r] == 0:
            per.append(0.0)
        else:
            per.append(math.inf)
            inf = True
    return per, (math.inf if inf else sum(per) / p)


def report_from_world(config: RunConfig, world: WorldReport) -> RunReport:
    """Totals of a run from its trace (P/src/bench.cpp:146-159)."""
    unit = 1e-9 if config.mode == "wall" else 1.0
    comp = sum(ev.t_end - ev.t_start for ev in world.trace if ev.kind == "compute") * unit
    over = sum(ev.t_end - ev.t_start for ev in world.trace if ev.kind != "compute") * unit
    return RunReport(config, world.wall_seconds if config.mode == "wall" else 0.0,
                     world.weighted_ops, comp, over, world)


def exp1_csv_row(r: RunReport) -> str:
    """One experiment-1 CSV row (P/src/bench.cpp:211-222)."""
    c = r.config
    return ",".join([c.algorithm, str(c.n), str(c.procs), str(c.cores),
                     format_double(r.wall_seconds), str(r.weighted_ops),
                     format_double(r.compute_total), format_double(r.overhead_total),
                     format_double(overhead_ratio(r.world)[1])])


def trace_to_jsonl(r: RunReport) -> str:
    """One compact JSON object per event (P/src/bench.cpp:335-350)."""
    rid = run_id(r.config)
    return "".join(json.dumps({"run_id": rid, "rank": ev.rank, "kind": ev.kind,
                               "t_start_ns": ev.t_start, "t_end_ns": ev.t_end,
                               "bytes": ev.bytes}, separators=(",", ":")) + "\n"
                   for ev in r.world.trace)


def trace_summary_json(r: RunReport) -> str:
    """Per-rank compute / communication / idle totals and counters, indented
    by 2 (P/src/bench.cpp:352-395)."""
    w = r.world
    p = w.procs
    comp, comm, idle = [0] * p, [0] * p, [0] * p
    for ev in w.trace:
        d = ev.t_end - ev.t_start
        if ev.kind == "compute":
            comp[ev.rank] += d
        elif ev.kind == "idle":
            idle[ev.rank] += d
        else:
            comm[ev.rank] += d
    ranks = []
    for i in range(p):
        cnt = w.counters[i] if i < len(w.counters) else {}
        ranks.append({"rank": i, "compute": comp[i], "communication": comm[i], "idle": idle[i],
                      "counters": {k: int(cnt.get(k, 0)) for k in _COUNTERS}})
    summary = {"run_id": run_id(r.config), "mode": r.config.mode, "procs": p,
               "cores": w.core_slots, "ranks": ranks}
    return json.dumps(summary, indent=2) + "\n"


def emit_trace(r: RunReport, path: str) -> None:
    """``path`` gets the JSONL, ``path + ".summary.json"`` the summary
    (P/src/bench.cpp:397-417)."""
    with open(path, "w") as f:
        f.write(trace_to_jsonl(r))
    with open(path + ".summary.json", "w") as f:
        f.write(trace_summary_json(r))


# ---------------------------------------------------------------------------
# GPU runs


def run_benchmark(config: RunConfig, ctx=None) -> RunReport:
    """bench::run_benchmark on one GPU (P/src/bench.cpp:106-169): gen_data's
    int64 stream on the device, the partitioned sort with one 'rank' per
    block (see the module docstring), each repetition verified on the device
    (sorted, and the multiset of the output equals the input's, else
    VerificationError), the median repetition reported (lower middle)."""
    import torch

    from .device import default_context
    if config.procs < 1 or config.cores < 1 or config.repetitions < 1:
        raise ConfigError(f"invalid run configuration: {config}")
    if config.algorithm not in ALGORITHMS:
        raise ConfigError(f"unknown algorithm '{config.algorithm}'")
    if config.mode != "wall":
        raise ConfigError("the GPU path has wall mode only (counted mode counts CPU operations)")
    ctx = ctx or default_context()
    from .sortbench import plan_partition
    n, p = config.n, config.procs
    data = ctx.gen_keys(n, config.seed, torch.int64)
    _, _, ms_in = ctx.check_sorted(data) if n else (0, 0, 0)
    sizes = plan_partition(n, p).sizes
    offs = [0]
    for s in sizes:
        offs.append(offs[-1] + s)
    rank_ctx = _rank_contexts(ctx, p)
    streams = [torch.cuda.Stream(ctx.device) for _ in range(p)]
    main = torch.cuda.current_stream(ctx.device)
    worlds = []
    for _ in range(config.repetitions):
        seg = torch.empty_like(data)
        out = torch.empty_like(data)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * p + 3)]
        ev[0].record(main)
        for r in range(p):  # every rank sorts its block on its own stream
            streams[r].wait_stream(main)
            ev[1 + 2 * r].record(streams[r])
            if sizes[r]:
                rank_ctx[r].sort(data[offs[r]:offs[r + 1]], out=seg[offs[r]:offs[r + 1]],
                                 stream=streams[r])
            ev[2 + 2 * r].record(streams[r])
        for r in range(p):
            main.wait_stream(streams[r])
        ev[2 * p + 1].record(main)
        runs = [seg[offs[r]:offs[r + 1]] for r in range(p) if sizes[r]]
        if runs:
            ctx.merge(runs, out=out, stream=main)
        ev[2 * p + 2].record(main)
        torch.cuda.synchronize(ctx.device)
        ns = [int(round(ev[0].elapsed_time(e) * 1e6)) for e in ev]
        if n:
            inv, _, ms_out = ctx.check_sorted(out)
            if inv != 0 or ms_out != ms_in:
                raise VerificationError(
                    f"run produced output that is not the sorted input: {config}")
        trace = []
        for r in range(p):
            trace.append(TraceEvent(r, "compute", ns[1 + 2 * r], ns[2 + 2 * r]))
        trace.append(TraceEvent(0, "gather", ns[2 * p + 1], ns[2 * p + 2], 8 * n))
        trace.sort(key=lambda e: (e.rank, e.t_start))
        counters = [{"element_moves": 0} for _ in range(p)]
        worlds.append(WorldReport(p, config.cores, "wall", ns[-1] * 1e-9, trace, counters))
    order = sorted(range(len(worlds)), key=lambda i: worlds[i].wall_seconds)
    return report_from_world(config, worlds[order[(len(order) - 1) // 2]])


_RANK_CTX: dict = {}


def _rank_contexts(ctx, p: int) -> list:
    """One context per rank on ctx's device (rank 0 is ctx itself), kept for
    later runs."""
    from .device import Context
    extra = _RANK_CTX.setdefault(ctx.device, [])
    while len(extra) < p - 1:
        extra.append(Context(ctx.device))
    return [ctx] + extra[:p - 1]


def experiment1(algorithms, n_per_algorithm, proc_list, core_list, seed: int = 1,
                repetitions: int = 1, ctx=None):
    """bench::experiment1 (P/src/bench.cpp:224-254) on the GPU: one verified
    report per (algorithm, m, k); returns (csv rows, reports)."""
    if not algorithms or not proc_list or not core_list:
        raise ConfigError("experiment 1 needs non-empty algorithm, process and core grids")
    if len(n_per_algorithm) != len(algorithms):
        raise ConfigError("experiment 1 needs one data size per algorithm")
    rows, reports = [], []
    for algo, n in zip(algorithms, n_per_algorithm):
        for m in proc_list:
            for k in core_list:
                rep = run_benchmark(RunConfig(algo, n, m, k, seed, "wall", repetitions), ctx)
                rows.append(exp1_csv_row(rep))
                reports.append(rep)
    return rows, reports


def run_benchmark_multi(config: RunConfig, devices: list, multi=None) -> RunReport:
    """bench::run_benchmark (P/src/bench.cpp:106-169) with procs = GPUs: the
    multi-GPU sample sort of the C ABI (b2s_sample_sort, one host thread per
    rank) on ``devices[:procs]`` (a repeated device emulates ranks on it).
    gen_data's int64 stream is generated shard by shard on each rank's device;
    every repetition is verified (concatenated buckets sorted, multiset equal
    to the input's); wall_seconds is the call's host wall time (the reference
    times its world from spawn to join, P/src/runtime.cpp:87,689). The trace
    has one compute (local sort), bcast (splitters) and gather (exchange +
    merge of the rank's bucket) event per rank, from rank 0's CUDA events."""
    import torch

    from .device import Context, MultiContext
    from .sortbench import plan_partition
    if config.procs < 1 or config.cores < 1 or config.repetitions < 1:
        raise ConfigError(f"invalid run configuration: {config}")
    if config.algorithm not in ALGORITHMS:
        raise ConfigError(f"unknown algorithm '{config.algorithm}'")
    p = config.procs
    if len(devices) < p:
        raise ConfigError(f"{p} ranks need {p} devices (got {devices})")
    devs = list(devices[:p])
    own = multi is None
    multi = multi or MultiContext(devs)
    sizes = plan_partition(config.n, p).sizes
    ctxs = {d: Context(d) for d in set(devs)}
    try:
        shards, off = [], 0
        for r in range(p):
            shards.append(ctxs[devs[r]].gen_keys(sizes[r], config.seed, torch.int64, first=off))
            off += sizes[r]
        ms_in = sum(ctxs[devs[r]].check_sorted(shards[r])[2] for r in range(p)) & ((1 << 64) - 1)
        worlds = []
        for _ in range(config.repetitions):
            buckets, _ = multi.sample_sort(shards)
            t = multi.timing()
            cat = torch.cat([b.to(f"cuda:{devs[0]}") for b in buckets])
            inv, _, ms_out = ctxs[devs[0]].check_sorted(cat) if cat.numel() else (0, 0, 0)
            if inv != 0 or (cat.numel() and ms_out != ms_in) or cat.numel() != config.n:
                raise VerificationError(f"run produced output that is not the sorted input: {config}")
            a = int(round(t.local_sort_ms * 1e6))
            b = a + int(round(t.splitters_ms * 1e6))
            c = b + int(round(t.exchange_merge_ms * 1e6))
            trace = []
            for r in range(p):
                trace += [TraceEvent(r, "compute", 0, a), TraceEvent(r, "bcast", a, b),
                          TraceEvent(r, "gather", b, c, 8 * buckets[r].numel())]
            counters = [{"element_moves": 0} for _ in range(p)]
            worlds.append(WorldReport(p, config.cores, "wall", t.total_ms * 1e-3, trace, counters))
        order = sorted(range(len(worlds)), key=lambda i: worlds[i].wall_seconds)
        return report_from_world(config, worlds[order[(len(order) - 1) // 2]])
    finally:
        for c in ctxs.values():
            c.close()
        if own:
            multi.close()


def trace_from_sample_sort(config: RunConfig, per_rank_phases: list, n_per_rank: list,
                           key_bytes: int = 4) -> RunReport:
    """A multi-GPU SampleSorter run as the reference's trace: per GPU rank,
    local sort -> compute, splitter selection (sample all-gather) -> bcast,
    exchange -> send, k-way merge -> compute. ``per_rank_phases[r]`` is that
    rank's ``SampleSorter.last_phase_ms`` (phases in order)."""
    trace = []
    kinds = {"local_sort": "compute", "splitters": "bcast", "exchange": "send", "merge": "compute"}
    wall = 0.0
    for r, phases in enumerate(per_rank_phases):
        t = 0
        for name, ms in phases.items():
            if name not in kinds:
                continue
            d = int(round(ms * 1e6))
            b = key_bytes * n_per_rank[r] if name == "exchange" else 0
            trace.append(TraceEvent(r, kinds[name], t, t + d, b))
            t += d
        wall = max(wall, t * 1e-9)
    p = len(per_rank_phases)
    world = WorldReport(p, config.cores, "wall", wall, trace, [{} for _ in range(p)])
    return report_from_world(config, world)
