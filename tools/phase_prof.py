"""Per-phase cycle split of the onesweep kernel (debug library from `make prof`).

  B2S_LIB=paper_1105_6040_b200/lib/libb200sort_prof.so python tools/phase_prof.py [n] [uni|zipf|asc|lo8|hi8]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1105_6040_b200 import _lib  # noqa: E402
from paper_1105_6040_b200.device import Context  # noqa: E402

NAMES = ["tma_wait+loop_top", "load+early_counts+sync", "digit_scan+sync", "rank",
         "lookback+sync", "writeout+sync", "-", "-"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
kind = sys.argv[2] if len(sys.argv) > 2 else "uni"
ctx = Context(0)
if kind == "zipf":
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from config_bench import zipf_keys
    keys = zipf_keys(ctx, n).view(torch.uint32)
elif kind == "lo8":  # one active digit: a keys-only sort runs it as the ticket pass
    keys = (ctx.gen_keys(n, 1, torch.uint32, shift=32).view(torch.int32) & 0xFF).view(torch.uint32)
elif kind == "hi8":  # one active digit behind a payload-free ... (top digit only)
    keys = (ctx.gen_keys(n, 1, torch.uint32, shift=32).view(torch.int32) & 0x7F000000).view(torch.uint32)
elif kind == "asc":
    keys = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
else:
    keys = ctx.gen_keys(n, 1, torch.uint32, shift=32)
out = torch.empty_like(keys)
ctx.sort(keys, out=out)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
_lib.lib().b2s_debug_phase_cycles(buf, 1)
ctx.sort(keys, out=out)
torch.cuda.synchronize()
_lib.lib().b2s_debug_phase_cycles(buf, 1)
tiles = (n + 12287) // 12288  # 512 x 24 u32 tiles
for who, off in (("thread 0 (look-back warp)", 0), ("last thread", 8)):
    tot = sum(buf[off + k] for k in range(8)) or 1
    print(who + ": " + ", ".join(f"{NAMES[k]} {100 * buf[off + k] / tot:.1f}%" for k in range(6)))
    print("   cycles per tile: " + ", ".join(f"{NAMES[k]} {buf[off + k] / tiles:.0f}" for k in range(6)))
