"""Single-GPU throughput of every BASELINE.json configuration's device work
(CUDA events, inputs resident in HBM, results checked on the device).

  python tools/config_bench.py [--out profiles/r01_configs.jsonl]

cfg1  N=2^20 int32 in [0,2^31), p=4: partitioned sort (scatter, 4 local
      sorts, merge) -- launch-latency bound at this size.
cfg2  N=2^28 uint32 full range: one local sort (the bench.py headline).
cfg3  per-GPU share of 2^31 int32 at G=8 (2^28 keys): local sort + the
      stable merge of 8 received runs (the exchange itself needs 8 GPUs).
cfg4  N=2^27 int32 on one GPU: (a) Zipf s=1.2 over 2^20 values, (b) sorted,
      (c) reverse, (d) all-equal.
cfg5  N=2^28 (uint64 key, uint32 index) pairs, stable.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1105_6040_b200.device import Context  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def zipf_keys(ctx, n, s=1.2, values=1 << 20, seed=1):
    """Zipf(s) over `values` ranks via inverse CDF of u = (z >> 11) * 2^-53 on the
    gen_data stream, rank -> value = rank."""
    z = ctx.gen_keys(n, seed, torch.int64).view(torch.int64)
    u = ((z >> 11) & ((1 << 53) - 1)).to(torch.float64) * (2.0 ** -53)
    w = torch.arange(1, values + 1, dtype=torch.float64, device=z.device) ** (-s)
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    return torch.searchsorted(cdf, u).clamp_(max=values - 1).to(torch.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ctx = Context(0)
    rows = []

    def record(cfg, name, n, ms, extra=None):
        row = {"config": cfg, "case": name, "n": n, "ms": ms, "keys_per_s": n / (ms * 1e-3)}
        row.update(extra or {})
        rows.append(row)
        print(json.dumps(row), flush=True)

    def sort_case(cfg, name, keys, vals=None, p=1):
        out = torch.empty_like(keys)
        vout = torch.empty_like(vals) if vals is not None else None
        if p == 1:
            fn = lambda: ctx.sort(keys, out=out, vals=vals, vals_out=vout)  # noqa: E731
        else:
            fn = lambda: ctx.partitioned_sort(keys, p, out=out, vals=vals, vals_out=vout)  # noqa: E731
        ms = timed(fn)
        ctx.enable_timing(True)
        fn()
        t = ctx.timing()
        ctx.enable_timing(False)
        inv, _, ms_out = ctx.check_sorted(out)
        _, _, ms_in = ctx.check_sorted(keys)
        assert inv == 0 and ms_in == ms_out, (cfg, name)
        kb = keys.element_size() + (4 if vals is not None else 0)
        gbs = [2 * kb * keys.numel() / (x * 1e-3) / 1e9 for x in t.pass_ms]
        record(cfg, name, keys.numel(), ms, {"passes_executed": t.passes_executed,
                                             "pass_ms": [round(x, 4) for x in t.pass_ms],
                                             "pass_gbs": [round(g) for g in gbs],
                                             "merge_ms": round(t.merge_ms, 4)})

    sort_case("cfg1", "N=2^20 i32 p=4 partitioned sort",
              ctx.gen_keys(1 << 20, 1, torch.int32, shift=33), p=4)
    # the reference's own p-phase algorithm on the device, same input
    k1 = ctx.gen_keys(1 << 20, 1, torch.int32, shift=33)
    o1 = torch.empty_like(k1)
    ms = timed(lambda: ctx.odd_even_sort(k1, 4, out=o1))
    inv, _, _ = ctx.check_sorted(o1)
    assert inv == 0
    record("cfg1", "N=2^20 i32 p=4 odd-even merge-split (the reference's algorithm on the GPU)",
           1 << 20, ms)
    sort_case("cfg2", "N=2^28 u32", ctx.gen_keys(1 << 28, 1, torch.uint32, shift=32))

    # cfg3 at G=1: all 2^31 int32 keys on one GPU (64-bit look-back words)
    big = ctx.gen_keys(1 << 31, 1, torch.int32, shift=33)
    sort_case("cfg3", "G=1: N=2^31 i32 on one GPU", big)
    del big
    torch.cuda.empty_cache()

    # cfg3 per-GPU work at G=8: local sort of a 2^28 shard + merge of 8 runs
    shard = ctx.gen_keys(1 << 28, 1, torch.int32, shift=33)
    sort_case("cfg3", "per-GPU local sort (2^28 i32 shard)", shard)
    # the 8 runs a GPU receives cover the same key range (each is one source's
    # slice of this bucket): sorted eighths of the random shard, interleaved
    runs = [ctx.sort(r.contiguous())[0] for r in torch.tensor_split(shard, 8)]
    mout = torch.empty_like(shard)
    ms = timed(lambda: ctx.merge(runs, out=mout))
    inv, _, _ = ctx.check_sorted(mout)
    assert inv == 0
    record("cfg3", "per-GPU merge of 8 received runs (2^28 i32, interleaved)", 1 << 28, ms,
           {"merge_gbs_per_round": round(3 * 8 * (1 << 28) / (ms * 1e-3) / 1e9)})
    del shard, runs, mout
    torch.cuda.empty_cache()

    n4 = 1 << 27
    sort_case("cfg4", "(a) Zipf s=1.2 over 2^20 values", zipf_keys(ctx, n4))
    sort_case("cfg4", "(b) ascending", torch.arange(n4, dtype=torch.int32, device="cuda"))
    sort_case("cfg4", "(c) descending", torch.arange(n4 - 1, -1, -1, dtype=torch.int32, device="cuda"))
    sort_case("cfg4", "(d) all equal", torch.full((n4,), 7, dtype=torch.int32, device="cuda"))

    n5 = 1 << 28
    sort_case("cfg5", "N=2^28 (u64 key, u32 index) stable",
              ctx.gen_keys(n5, 1, torch.uint64), torch.arange(n5, dtype=torch.int32, device="cuda"))
    if a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    ctx.close()


if __name__ == "__main__":
    main()
