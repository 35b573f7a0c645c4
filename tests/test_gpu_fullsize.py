"""GPU: every BASELINE.json configuration at its FULL size, generated on the
device from the same seeded stream as tests/golden/make_fullsize.py, sorted
through the C ABI and compared with the CPU-computed fingerprint of the
expected output (the reference's gate is std::sort equality,
P/src/bench.cpp:95-104; the fingerprint is order-sensitive over every
position, so a mismatch anywhere fails). The input's multiset hash is checked
too, so a generator drift cannot pass as a sort error or vice versa."""
import json
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1105_6040_b200 import workloads  # noqa: E402
from paper_1105_6040_b200.device import Context  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = {c["config"]: c for c in json.load(open(os.path.join(HERE, "golden", "fullsize.json")))["configs"]}


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()
    torch.cuda.empty_cache()


def _check(ctx, name, keys, out):
    g = GOLD[name]
    assert keys.numel() == g["n"]
    _, _, ms_in = ctx.check_sorted(keys)
    assert ms_in == int(g["input_multiset"]), f"{name}: input differs from the golden input"
    inv, fp, ms = ctx.check_sorted(out)
    assert inv == 0, f"{name}: {inv} adjacent inversions"
    assert ms == int(g["multiset"]), f"{name}: output is not a permutation of the input"
    assert fp == int(g["fp"]), f"{name}: output differs from the expected sorted array"


def test_cfg2_full(ctx):
    keys = ctx.gen_keys(1 << 28, 1, torch.uint32, shift=32)
    out, _ = ctx.sort(keys)
    _check(ctx, "cfg2", keys, out)


@pytest.mark.parametrize("p", [1, 8])
def test_cfg3_full_one_gpu(ctx, p):
    """2^31 int32 keys on one GPU: the plain sort (p=1) and the partitioned
    sort with 8 partitions (8 local sorts + the root merge at full size)."""
    keys = ctx.gen_keys(1 << 31, 1, torch.int32, shift=33)
    out = torch.empty_like(keys)
    if p == 1:
        ctx.sort(keys, out=out)
    else:
        ctx.partitioned_sort(keys, p, out=out)
    _check(ctx, "cfg3", keys, out)
    del keys, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kind,name", [("zipf", "cfg4a"), ("ascending", "cfg4b"),
                                       ("descending", "cfg4c"), ("equal", "cfg4d")])
def test_cfg4_full(ctx, kind, name):
    keys = workloads.cfg4_keys(ctx, kind, 1 << 27)
    out, _ = ctx.sort(keys)
    _check(ctx, name, keys, out)
    out8, _ = ctx.partitioned_sort(keys, 8)
    _check(ctx, name, keys, out8)


def test_cfg4a_thresholds_pinned():
    import oracle
    t = workloads.zipf_thresholds()
    assert str(oracle.fingerprint(t)) == GOLD["cfg4a"]["thresholds_fp"]


def test_cfg5_full(ctx):
    """2^28 (uint64 key, uint32 original index) pairs: keys AND the payload
    permutation equal the stable order."""
    n = 1 << 28
    keys = ctx.gen_keys(n, 1, torch.uint64)
    vals = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    ok, ov = ctx.sort(keys, vals=vals)
    _check(ctx, "cfg5", keys, ok)
    _, vfp, _ = ctx.check_sorted(ov)
    assert vfp == int(GOLD["cfg5"]["payload_fp"]), "cfg5: payload order differs from the stable order"


@pytest.mark.parametrize("n", [3 << 29, 1 << 31])
def test_narrow_lookback_words_past_2_30(ctx, n):
    """Between 2^30 and 2^31 keys the look-back words stay 32-bit and hold
    prefixes modulo 2^30 (radix_sort.cu narrow_lookback_words). A digit with
    more than 2^30 keys makes its prefixes wrap: 3 keys in 4 get low byte 7
    (the skewed pass), so the first pass resolves prefixes past 2^30."""
    keys = ctx.gen_keys(n, 5, torch.int32, shift=32)
    hot = ((keys >> 8) & 3) != 0
    keys = torch.where(hot, (keys & ~0xFF) | 7, keys)
    del hot
    _, _, ms_in = ctx.check_sorted(keys)
    out = torch.empty_like(keys)
    ctx.sort(keys, out=out)
    inv, _, ms = ctx.check_sorted(out)
    assert inv == 0, f"{inv} adjacent inversions"
    assert ms == ms_in, "output is not a permutation of the input"
    del keys, out
    torch.cuda.empty_cache()


def test_wide_lookback_words_past_2_31(ctx):
    """Above 2^31 keys the look-back words are 64-bit (the only sizes that
    still use them): a sort of 2^31 + 3 * 2^20 + 7 int32 keys, with a
    partial last tile, checked by order and multiset."""
    n = (1 << 31) + 3 * (1 << 20) + 7
    keys = ctx.gen_keys(n, 9, torch.int32, shift=32)
    _, _, ms_in = ctx.check_sorted(keys)
    out = torch.empty_like(keys)
    ctx.sort(keys, out=out)
    inv, _, ms = ctx.check_sorted(out)
    assert inv == 0, f"{inv} adjacent inversions"
    assert ms == ms_in, "output is not a permutation of the input"
    del keys, out
    torch.cuda.empty_cache()
