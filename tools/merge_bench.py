"""k-way merge throughput on one GPU: k sorted runs of an n-key array (the
per-GPU merge of cfg3), CUDA events, inputs resident.
  python tools/merge_bench.py [n] [k ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1105_6040_b200.device import Context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
ks = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
dt = torch.uint64 if os.environ.get("MERGE_DTYPE") == "u64" else torch.int32
ctx = Context(0)
keys = ctx.gen_keys(n, 1, dt, shift=33 if dt == torch.int32 else 0)
for k in ks:
    runs = [ctx.sort(r.contiguous())[0] for r in torch.tensor_split(keys, k)]
    out = torch.empty_like(keys)
    for _ in range(2):
        ctx.merge(runs, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        ctx.merge(runs, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    inv, _, _ = ctx.check_sorted(out)
    rounds = max(1, (k - 1).bit_length())
    kb = keys.element_size()
    print(f"k={k} n={n} {ms:.3f} ms, {rounds} rounds, {rounds * 2 * kb * n / (ms * 1e-3) / 1e9:.0f} GB/s "
          f"per-round algorithmic, sorted={inv == 0}", flush=True)
    del runs, out
