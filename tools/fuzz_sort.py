"""Randomised differential test of the sort (and k-way merge) against
torch.sort on the same GPU, for a fixed wall-clock budget: log-uniform sizes
up to 2^26 (every tile configuration, partial tiles, the twin kernels),
every key type, distributions from uniform to all-equal -- among them the
inputs of the adaptive paths: presorted with and without one swapped pair or
duplicates, and 8-byte keys whose upper halves tie in runs of every length --
with and without a payload (checked against torch's stable order), in and out
of place. A third of the cases are drawn from 2^20..2^25 keys, where those
paths apply.

  python tools/fuzz_sort.py [seconds] [seed]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1105_6040_b200.device import Context  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ctx = Context(0)
DT = [torch.int32, torch.uint32, torch.int64, torch.uint64]
SIGNED = {torch.uint32: torch.int32, torch.uint64: torch.int64}


def as_signed_order(t):
    """Keys mapped to a signed tensor with the same order (torch.sort has no
    unsigned sort)."""
    if t.dtype in SIGNED:
        s = t.view(SIGNED[t.dtype])
        flip = torch.tensor(-(1 << (8 * t.element_size() - 1)), dtype=s.dtype, device=t.device)
        return s ^ flip
    return t


def make(n, dt, kind):
    bits = 8 * torch.empty(0, dtype=dt).element_size()
    seed = int(rng.integers(1 << 30))
    k = ctx.gen_keys(n, seed, torch.int64 if bits == 64 else torch.int32, shift=0 if bits == 64 else 32)
    if kind == "few":
        k = k & 0x7
    elif kind == "bytes":  # a few varying bytes
        k = k & (0x00FF00FF if bits == 32 else 0x00FF0000000000FF)
    elif kind == "asc":
        k = torch.arange(n, device="cuda", dtype=k.dtype)
    elif kind == "desc":
        k = torch.arange(n, 0, -1, device="cuda", dtype=k.dtype)
    elif kind == "equal":
        k = torch.full((n,), -3, device="cuda", dtype=k.dtype)
    elif kind == "hot":  # one digit value for most keys
        k = torch.where((k & 0xF) != 0, k & ~0xFF, k)
    elif kind in ("asc_swap", "desc_swap"):  # presorted but for one pair
        k = torch.arange(n, device="cuda", dtype=k.dtype) if kind == "asc_swap" else \
            torch.arange(n, 0, -1, device="cuda", dtype=k.dtype)
        if n > 1:
            i = int(rng.integers(n - 1))
            k[i:i + 2] = k[i:i + 2].flip(0)
    elif kind == "desc_dups":  # non-increasing with equal neighbours
        k = (torch.arange(n, 0, -1, device="cuda", dtype=k.dtype) >> 2)
    elif kind == "sorted_rand":  # ascending random keys (signed: crossing zero)
        k = torch.sort(k)[0]
        if rng.integers(2):
            k = k.flip(0)
    elif kind == "upper_ties" and bits == 64:
        # upper halves drawn from a pool: tie runs of ~2 .. ~n/4 keys; lower
        # halves random, few-valued or constant
        pool = max(1, n // int(2 ** rng.integers(1, 14)))
        idx = torch.randint(0, pool, (n,), device="cuda")
        hi = (idx * 0x9E3779B1 + 12345) & 0xFFFFFFFF
        lo = [k & 0xFFFFFFFF, k & 0x3, torch.zeros_like(k)][int(rng.integers(3))]
        k = (hi << 32) | lo
    return k.view(dt) if dt in SIGNED else k.to(dt)


t0 = time.time()
cases = 0
while time.time() - t0 < budget:
    if rng.integers(3) == 0:
        n = int(np.exp(rng.uniform(np.log(1 << 20), np.log(1 << 25))))
    else:
        n = int(np.exp(rng.uniform(0, np.log(1 << 26))))
    dt = DT[int(rng.integers(4))]
    kinds = ["uniform", "few", "bytes", "asc", "desc", "equal", "hot", "asc_swap", "desc_swap",
             "desc_dups", "sorted_rand", "upper_ties"]
    kind = kinds[int(rng.integers(len(kinds)))]
    keys = make(n, dt, kind)
    ref_k, ref_i = torch.sort(as_signed_order(keys), stable=True)
    in_place = bool(rng.integers(2))
    if rng.integers(2):
        vals = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
        if in_place:
            ok, ov = keys.clone(), vals
            ctx.sort(ok, out=ok, vals=ov, vals_out=ov)
        else:
            ok, ov = ctx.sort(keys, vals=vals)
        good = torch.equal(as_signed_order(ok), ref_k) and \
            torch.equal(ov.view(torch.int32).to(torch.int64), ref_i)
    else:
        if in_place:
            ok = keys.clone()
            ctx.sort(ok, out=ok)
        else:
            ok, _ = ctx.sort(keys)
        good = torch.equal(as_signed_order(ok), ref_k)
    if not good:
        print(f"MISMATCH n={n} dtype={dt} kind={kind} in_place={in_place}", flush=True)
        sys.exit(1)
    if rng.integers(4) == 0 and n > 8:  # k-way merge of sorted pieces
        k = int(rng.integers(2, 17))
        runs = [ctx.sort(r.contiguous())[0] for r in torch.tensor_split(keys, k)]
        mk, _ = ctx.merge(runs)
        if not torch.equal(as_signed_order(mk), ref_k):
            print(f"MERGE MISMATCH n={n} k={k} dtype={dt} kind={kind}", flush=True)
            sys.exit(1)
    cases += 1
    del keys, ref_k, ref_i
print(f"fuzz ok: {cases} cases in {time.time() - t0:.0f} s", flush=True)
