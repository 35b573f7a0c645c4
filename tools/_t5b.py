import sys, torch
sys.path.insert(0, '.')
from paper_1105_6040_b200.device import Context
ctx = Context(0)
n = 1 << 28
keys = ctx.gen_keys(n, 1, torch.uint64, shift=0)
vals = torch.arange(n, dtype=torch.int32, device='cuda').view(torch.uint32)
ok = torch.empty_like(keys); ov = torch.empty_like(vals)
for i in range(2):
    ctx.sort(keys, out=ok, vals=vals, vals_out=ov)
torch.cuda.synchronize()
