"""cfg1 (2^20 int32, p = 4 partitioned sort) per-call time with and without the
captured CUDA graph: GPU time per call, host enqueue time and single-call wall
latency.   python tools/graph_bench.py ; B2S_GRAPHS=0 python tools/graph_bench.py"""
import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1105_6040_b200.device import Context
ctx = Context(0)
n, p = 1 << 20, 4
keys = ctx.gen_keys(n, 1, torch.int32, shift=33)
out = torch.empty_like(keys)
for _ in range(3):
    ctx.partitioned_sort(keys, p, out=out)
torch.cuda.synchronize()
for reps in (5, 50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        ctx.partitioned_sort(keys, p, out=out)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(os.environ.get("B2S_GRAPHS", "1"), reps, "gpu ms/call", e0.elapsed_time(e1) / reps, "host enqueue ms/call", (t1 - t0) * 1e3 / reps, "wall", (t2 - t0) * 1e3 / reps)
# single call latency
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.partitioned_sort(keys, p, out=out)
    torch.cuda.synchronize()
    print("single call wall ms", (time.perf_counter() - t0) * 1e3)
