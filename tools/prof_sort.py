"""Small driver for kernel timing / ncu captures of the radix passes.

  python tools/prof_sort.py --n 67108864 --dtype u32 --iters 3 [--vals]
Prints one line per iteration with the per-phase CUDA-event times.
Tile configurations are build switches (B2S_U32_ITEMS; tools/kdev_build.sh).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1105_6040_b200.device import Context  # noqa: E402

DT = {"u32": (torch.uint32, 32), "i32": (torch.int32, 33), "u64": (torch.uint64, 0),
      "i64": (torch.int64, 0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 26)
    ap.add_argument("--dtype", default="u32")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--vals", action="store_true")
    ap.add_argument("--merge-k", type=int, default=0)
    a = ap.parse_args()
    ctx = Context(0)
    dt, shift = DT[a.dtype]
    keys = ctx.gen_keys(a.n, 1, dt, shift=shift)
    out = torch.empty_like(keys)
    vals = torch.arange(a.n, dtype=torch.int32, device="cuda") if a.vals else None
    vout = torch.empty_like(vals) if a.vals else None
    ctx.enable_timing(True)
    kb = keys.element_size() + (4 if a.vals else 0)
    for i in range(a.iters):
        if a.merge_k:
            srt, _ = ctx.sort(keys)
            runs = list(torch.tensor_split(srt, a.merge_k))
            runs = [ctx.sort(r.contiguous())[0] for r in runs]
            ctx.merge(runs, out=out)
            t = ctx.timing()
            gbs = 2 * keys.element_size() * a.n * t.merge_rounds / (t.merge_ms * 1e-3) / 1e9
            print(f"iter {i}: merge k={a.merge_k} rounds={t.merge_rounds} {t.merge_ms:.3f} ms "
                  f"({gbs:.0f} GB/s per round avg)", flush=True)
            continue
        ctx.sort(keys, out=out, vals=vals, vals_out=vout)
        t = ctx.timing()
        passes = " ".join(f"{p:.3f}" for p in t.pass_ms)
        gbs = [2 * kb * a.n / (p * 1e-3) / 1e9 for p in t.pass_ms]
        print(f"iter {i}: hist {t.hist_ms:.3f} ms ({kb * a.n / (t.hist_ms * 1e-3) / 1e9:.0f} GB/s)"
              f" passes[{t.passes_executed}] {passes} ms -> "
              + " ".join(f"{g:.0f}" for g in gbs) + " GB/s"
              f" copy {t.copy_ms:.3f} total {t.total_ms:.3f} ms", flush=True)
    inv, _, _ = ctx.check_sorted(out)
    assert inv == 0
    ctx.close()


if __name__ == "__main__":
    main()
