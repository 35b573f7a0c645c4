"""Bucket balance of the multi-GPU sample sort on every BASELINE config
("report max/min bucket size per config"), through the C ABI
(b2s_sample_sort) with G ranks emulated on one device (or real devices with
--devices). Each shard is plan_partition's slice of the config's stream; the
buckets are checked for order within and across ranks and for the multiset.
Emulated ranks run one after another on one GPU, so the phase times are not
multi-GPU timings; the balance is exact.

  python tools/multi_balance.py [--devices 0,0,0,0,0,0,0,0] > profiles/r02_multi_balance.jsonl
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1105_6040_b200 import workloads  # noqa: E402
from paper_1105_6040_b200.device import Context, MultiContext  # noqa: E402


def plan(n, p):
    q, r = divmod(n, p)
    return [q + (1 if i < r else 0) for i in range(p)]


def run(mc, ctx, name, shards, vals=None):
    G = len(shards)
    buckets, bvals = mc.sample_sort(shards, vals=vals)
    t = mc.timing()
    ms_in = sum(ctx.check_sorted(s)[2] for s in shards) & ((1 << 64) - 1)
    ms_out, inv, prev = 0, 0, None
    for b in buckets:
        i, _, m = ctx.check_sorted(b)
        inv += i
        ms_out = (ms_out + m) & ((1 << 64) - 1)
        if b.numel():
            first = b[0].item()
            if prev is not None and first < prev:
                inv += 1
            prev = b[-1].item()
    sizes = [b.numel() for b in buckets]
    n = sum(sizes)
    rec = {"config": name, "ranks": G, "n": n, "max_bucket": max(sizes), "min_bucket": min(sizes),
           "max_over_mean": max(sizes) * G / n, "bucket_sizes": sizes,
           "sorted": inv == 0, "permutation": ms_in == ms_out, "transport": t.transport,
           "phase_ms_emulated": {"local_sort": t.local_sort_ms, "splitters": t.splitters_ms,
                                 "exchange_merge": t.exchange_merge_ms}}
    if vals is not None:
        # payload = original index: stable iff equal keys carry ascending indices
        ok = True
        for b, v in zip(buckets, bvals):
            if b.numel() > 1:
                k64 = b.view(torch.int64) if b.dtype == torch.uint64 else b.to(torch.int64)
                same = k64[1:] == k64[:-1]
                vv = v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
                ok &= bool((~same | (vv[1:] > vv[:-1])).all())
        rec["stable"] = ok
    print(json.dumps(rec), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--devices", default="0,0,0,0,0,0,0,0")
    ap.add_argument("--skip-cfg3", action="store_true")
    args = ap.parse_args()
    devs = [int(d) for d in args.devices.split(",")]
    G = len(devs)
    ctx = Context(devs[0])
    mc = MultiContext(devs)
    if not args.skip_cfg3:
        n = 1 << 31
        offs = [0]
        for s in plan(n, G):
            offs.append(offs[-1] + s)
        shards = [ctx.gen_keys(offs[r + 1] - offs[r], 1, torch.int32, shift=33, first=offs[r])
                  for r in range(G)]
        run(mc, ctx, "cfg3", shards)
        del shards
        torch.cuda.empty_cache()
    n = 1 << 27
    offs = [0]
    for s in plan(n, G):
        offs.append(offs[-1] + s)
    for kind, name in (("zipf", "cfg4a"), ("ascending", "cfg4b"), ("descending", "cfg4c"),
                       ("equal", "cfg4d")):
        shards = [workloads.cfg4_keys(ctx, kind, offs[r + 1] - offs[r], first=offs[r], total=n)
                  for r in range(G)]
        run(mc, ctx, name, shards)
        del shards
        torch.cuda.empty_cache()
    n = 1 << 28
    offs = [0]
    for s in plan(n, G):
        offs.append(offs[-1] + s)
    shards = [ctx.gen_keys(offs[r + 1] - offs[r], 1, torch.uint64, first=offs[r]) for r in range(G)]
    vals = [torch.arange(offs[r], offs[r + 1], dtype=torch.int64, device=f"cuda:{devs[r]}")
            .to(torch.int32).view(torch.uint32) for r in range(G)]
    run(mc, ctx, "cfg5", shards, vals)
    mc.close()
    ctx.close()


if __name__ == "__main__":
    main()
