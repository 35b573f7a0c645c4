"""Per-phase cycle split of the pipelined onesweep kernel (debug library built
with -DB2S_PHASE_PROFILE, e.g. `bash tools/kdev_build.sh prof -DB2S_PHASE_PROFILE`).

  B2S_LIB=paper_1105_6040_b200/lib/libb200sort_prof.so python tools/pipe_prof.py [n] [uni|asc]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1105_6040_b200 import _lib  # noqa: E402
from paper_1105_6040_b200.device import Context  # noqa: E402

NAMES = ["E tma wait", "E rank", "B1", "D digits", "K look-back", "reload+B2", "scatter+B3", "W store+B4"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
kind = sys.argv[2] if len(sys.argv) > 2 else "uni"
tile = int(os.environ.get("PIPE_TILE", 512 * 21))
ctx = Context(0)
if kind == "asc":
    keys = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
elif kind == "lo8":
    keys = (ctx.gen_keys(n, 1, torch.uint32, shift=32).view(torch.int32) & 0xFF).view(torch.uint32)
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
passes = 1 if kind == "lo8" else 4
tiles = passes * ((n + tile - 1) // tile)
for who, off in (("thread 0", 0), ("thread 511", 8)):
    tot = sum(buf[off + k] for k in range(8)) or 1
    print(who + f" ({tot / tiles:.0f} cycles per tile): " +
          ", ".join(f"{NAMES[k]} {buf[off + k] / tiles:.0f}" for k in range(8)))
