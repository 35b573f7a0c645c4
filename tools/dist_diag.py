"""Per-pass times of one distribution (diagnostics): python tools/dist_diag.py zipf|asc|uni"""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch  # noqa: E402

from config_bench import timed, zipf_keys  # noqa: E402
from paper_1105_6040_b200.device import Context  # noqa: E402

ctx = Context(0)
kind = sys.argv[1]
n = 1 << 27
if kind == "zipf":
    k = zipf_keys(ctx, n)
elif kind == "equal":
    k = torch.full((n,), 7, dtype=torch.int32, device="cuda")
elif kind == "asc":
    k = torch.arange(n, dtype=torch.int32, device="cuda")
else:
    k = ctx.gen_keys(n, 1, torch.int32, shift=32)
out = torch.empty_like(k)
ms = timed(lambda: ctx.sort(k, out=out))
ctx.enable_timing(True)
ctx.sort(k, out=out)
t = ctx.timing()
ctx.enable_timing(False)
print(kind, os.environ.get("B2S_LIB", "default").split("/")[-1], os.environ.get("B2S_SKEW_SHIFT"),
      round(ms, 4), "hist", round(t.hist_ms, 4), "copy", round(t.copy_ms, 4), [round(x, 4) for x in t.pass_ms])
