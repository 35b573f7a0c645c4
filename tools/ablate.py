"""Time one pass of each ablated onesweep build (output is wrong by design)."""
import os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for name in ["", "LOOKBACK", "RANK", "WRITE", "SCATTER", "NEXTHIST"]:
    env = dict(os.environ)
    if name:
        env["B2S_LIB"] = os.path.join(root, "paper_1105_6040_b200", "lib", f"libb200sort_lb{name}.so")
    code = ("import sys; sys.path.insert(0, %r)\n" % root) + '''
import torch
from paper_1105_6040_b200.device import Context
ctx = Context(0); n = 1 << 28
keys = ctx.gen_keys(n, 1, torch.uint32, shift=32); out = torch.empty_like(keys)
ctx.enable_timing(True)
ps = []
for i in range(4):
    ctx.sort(keys, out=out); t = ctx.timing(); ps += t.pass_ms[:1]
print(sum(ps[1:]) / len(ps[1:]))
'''
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"{name or 'full':10s} pass ms {r.stdout.strip()} {r.stderr.strip()[-200:]}")
