"""Sort check of one onesweep tile configuration (B2S_ONESWEEP_CFG): 2^26,
2^20 + 777 and 5000 uint32 keys against torch.sort. Used by
tests/test_gpu_rank_modes.py for every experimental configuration."""
import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_1105_6040_b200.device import Context
ctx = Context(0)
for n in (1 << 26, (1 << 20) + 777, 5000):
    k = ctx.gen_keys(n, 3, torch.uint32, shift=32)
    out, _ = ctx.sort(k)
    ref = torch.sort(k.view(torch.int32).to(torch.int64) & 0xFFFFFFFF)[0]
    ok = torch.equal(out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, ref)
    print(os.environ.get("B2S_ONESWEEP_CFG"), n, "OK" if ok else "MISMATCH", flush=True)
