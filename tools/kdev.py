"""A/B timing of onesweep development builds (u32 keys only).

  python tools/kdev.py lib1.so [VAR=1,lib2.so ...]      (on the GPU box)

Each library runs in its own process (B2S_LIB): uniform, Zipf-like and
ascending 2^28 u32 sorts, checked against torch.sort, reporting the average
pass time and the whole sort. Development builds come from
`bash tools/kdev_build.sh NAME "-DFOO=1"` (u32 default path only, ~20 s).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = '''
import sys, torch
sys.path.insert(0, %r)
from paper_1105_6040_b200.device import Context
ctx = Context(0); n = 1 << 28
res = []
import os
for kind in os.environ.get("KDEV_KINDS", "uni,skew,asc").split(","):
    if kind == "lo8":   # one active digit: a single pass (ablation builds write wrong output)
        keys = (ctx.gen_keys(n, 1, torch.uint32, shift=32).view(torch.int32) & 0xFF).view(torch.uint32)
    elif kind == "uni":
        keys = ctx.gen_keys(n, 1, torch.uint32, shift=32)
    elif kind == "skew":
        k = ctx.gen_keys(n, 2, torch.uint32, shift=32).view(torch.int32)
        keys = (k & (k >> 3) & (k >> 7)).view(torch.uint32)   # bits biased to 0: skewed digits
    else:
        # ascending but for one swapped pair, so the passes (structured twin)
        # run instead of the presorted shortcut
        k = torch.arange(n, dtype=torch.int32, device="cuda")
        k[:2] = torch.tensor([1, 0], dtype=torch.int32, device="cuda")
        keys = k.view(torch.uint32)
    out = torch.empty_like(keys)
    ctx.enable_timing(True)
    ps, tot = [], []
    for i in range(6):
        ctx.sort(keys, out=out)
        t = ctx.timing()
        if i >= 2:
            ps += t.pass_ms
            tot.append(t.total_ms)
    ref = torch.sort(keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF)[0]
    ok = bool(torch.equal(out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, ref))
    torch.cuda.synchronize()
    res.append("%%s pass %%.4f total %%.4f %%s" %% (kind, sum(ps) / len(ps), sum(tot) / len(tot), "OK" if ok else "MISMATCH"))
    del keys, out, ref
    torch.cuda.empty_cache()
print(" | ".join(res))
'''


def main():
    for arg in sys.argv[1:]:
        env = dict(os.environ)
        *sets, lib = arg.split(",")  # optional VAR=VALUE settings before the library
        for kv in sets:
            k, v = kv.split("=", 1)
            env[k] = v
        env["B2S_LIB"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, "-c", CODE % ROOT], env=env, capture_output=True, text=True)
        tail = r.stdout.strip() or r.stderr.strip()[-400:]
        print(f"{','.join(sets + [os.path.basename(lib)]):40s} {tail}", flush=True)


if __name__ == "__main__":
    main()
