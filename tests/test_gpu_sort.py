"""GPU: the onesweep radix sort (b2s_sort) against the oracle's merge-sort
restatement -- bit-exact for every key width, size class and distribution the
reference tests touch (empty, ragged tiles, duplicates, all-equal, sorted,
reverse, signed extremes) plus stability of the uint32 payload."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1105_6040_b200.device import Context  # noqa: E402

DTYPES = [np.int32, np.uint32, np.int64, np.uint64]
TORCH = {np.int32: torch.int32, np.uint32: torch.uint32, np.int64: torch.int64,
         np.uint64: torch.uint64}
# tile edges of every configuration: 512x20 (u32), 512x10 (u32+payload),
# 512x8 (u64), 512x6 (u64+payload), plus look-back word width edges elsewhere
SIZES = [0, 1, 2, 31, 1000, 3071, 3072, 3073, 4095, 4096, 4097, 5119, 5120, 5121, 8191, 8192,
         8193, 10239, 10240, 10241, 20480, 20481, 100_000, (1 << 20) + 7]


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


def rand_keys(n, dt, rng, kind="uniform"):
    info = np.iinfo(dt)
    if kind == "uniform":
        return rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    if kind == "dups":
        return rng.integers(0, 32, n).astype(dt)
    if kind == "equal":
        return np.full(n, info.max // 3, dtype=dt)
    if kind == "sorted":
        return np.sort(rng.integers(info.min, info.max, n, dtype=dt, endpoint=True))
    if kind == "reverse":
        return np.sort(rng.integers(info.min, info.max, n, dtype=dt, endpoint=True))[::-1].copy()
    if kind == "topbyte":
        shift = np.dtype(dt).itemsize * 8 - 8
        return (rng.integers(0, 256, n).astype(np.uint64) << np.uint64(shift)).astype(dt)
    if kind == "lowzero":  # digit 0 constant: the first active digit is recounted
        return (rng.integers(info.min, info.max, n, dtype=dt, endpoint=True) & ~dt(0xFF)).astype(dt)
    if kind == "midconst":  # a constant digit between varying ones
        ut = np.uint32 if np.dtype(dt).itemsize == 4 else np.uint64
        shift = ut(np.dtype(dt).itemsize * 8 - 16)
        x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True).view(ut)
        return (x & ~(ut(0xFF) << shift)).view(dt)
    if kind == "skewed":  # ~60% zeros: passes whose top digit is hot rank by ballots
        x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        return np.where(rng.random(n) < 0.6, dt(0), x).astype(dt)
    if kind == "extremes":
        return rng.choice(np.array([info.min, info.max, 0, 1, info.max - 1, info.min + 1],
                                   dtype=dt), n)
    raise ValueError(kind)


def to_dev(x):
    return torch.from_numpy(x).cuda() if x.dtype not in (np.uint32, np.uint64) else \
        torch.from_numpy(x.view(np.int32 if x.dtype == np.uint32 else np.int64)).cuda().view(
            TORCH[x.dtype.type])


def to_host(t, dt):
    if dt in (np.uint32, np.uint64):
        return t.view(torch.int32 if dt == np.uint32 else torch.int64).cpu().numpy().view(dt)
    return t.cpu().numpy()


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("n", SIZES)
def test_sort_uniform_sizes(ctx, dt, n):
    rng = np.random.default_rng(n * 7 + np.dtype(dt).itemsize)
    keys = rand_keys(n, dt, rng)
    out, _ = ctx.sort(to_dev(keys))
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out, dt), oracle.sort(keys))


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("kind", ["dups", "equal", "sorted", "reverse", "topbyte", "extremes",
                                  "lowzero", "midconst", "skewed"])
def test_sort_distributions(ctx, dt, kind):
    rng = np.random.default_rng(5)
    for n in (5000, 70_001):
        keys = rand_keys(n, dt, rng, kind)
        out, _ = ctx.sort(to_dev(keys))
        torch.cuda.synchronize()
        assert np.array_equal(to_host(out, dt), oracle.sort(keys)), (kind, n)


@pytest.mark.parametrize("dt", DTYPES)
def test_sort_in_place_and_host_buffers(ctx, dt):
    rng = np.random.default_rng(9)
    for kind in ("uniform", "topbyte", "dups", "equal"):  # 4/8, 1, 1 and 0 executed passes
        keys = rand_keys(50_000, dt, rng, kind)
        expect = oracle.sort(keys)
        d = to_dev(keys)
        ctx.sort(d, out=d)                      # device, in place
        torch.cuda.synchronize()
        assert np.array_equal(to_host(d, dt), expect), kind
        h = keys.copy()
        ctx.sort(h, out=h)                      # host buffers (B2S_HOST)
        assert np.array_equal(h, expect), kind
        before = keys.copy()
        h2, _ = ctx.sort(keys)                  # host, out of place
        assert np.array_equal(h2, expect) and np.array_equal(keys, before)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("kind", ["equal", "topbyte", "uniform", "dups"])
@pytest.mark.parametrize("n", [5000, 300_000, 5_000_000])
def test_sort_pairs_mixed_aliasing(ctx, dt, kind, n):
    """Keys sorted in place with the payload in a separate buffer, and the
    reverse: all-equal keys execute 0 passes, topbyte keys 1 (an odd count), so
    both exercise the trailing-copy and buffer-chain corner cases."""
    rng = np.random.default_rng(n + 3)
    keys = rand_keys(n, dt, rng, kind)
    vals = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    ek, ev = oracle.stable_sort_kv(keys, vals)
    tv = lambda x: torch.from_numpy(x.view(np.int32)).cuda()  # noqa: E731
    # keys in place, payload out of place
    dk, dv = to_dev(keys), tv(vals)
    dvo = torch.full_like(dv, -1)
    ctx.sort(dk, out=dk, vals=dv, vals_out=dvo)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(dk, dt), ek)
    assert np.array_equal(dvo.cpu().numpy().view(np.uint32), ev)
    # keys out of place, payload in place
    dk, dv = to_dev(keys), tv(vals)
    dko = torch.empty_like(dk)
    ctx.sort(dk, out=dko, vals=dv, vals_out=dv)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(dko, dt), ek)
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), ev)
    assert np.array_equal(to_host(dk, dt), keys)  # input keys untouched


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("kind", ["dups", "uniform", "equal", "skewed", "sorted", "reverse"])
@pytest.mark.parametrize("n", [123_457, 3072, 5121, 1, 8191, 8192, 8193, 16385])
def test_sort_pairs_stable(ctx, dt, kind, n):
    rng = np.random.default_rng(17)
    keys = rand_keys(n, dt, rng, kind)
    vals = np.arange(n, dtype=np.uint32)
    ek, ev = oracle.stable_sort_kv(keys, vals)
    ok, ov = ctx.sort(to_dev(keys), vals=torch.from_numpy(vals.view(np.int32)).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(to_host(ok, dt), ek)
    assert np.array_equal(ov.cpu().numpy().view(np.uint32), ev)
    # host path with payload
    hk, hv = ctx.sort(keys, vals=vals)
    assert np.array_equal(hk, ek) and np.array_equal(hv, ev)


def test_constant_digits_are_skipped(ctx):
    """int64 keys in [0, 2^31) (the reference's widened i32 data) run 4 of 8 passes."""
    ctx.enable_timing(True)
    try:
        z = oracle.gen_data(1 << 18, 1).view(np.uint64)
        keys = (z >> np.uint64(33)).astype(np.int64)
        out, _ = ctx.sort(to_dev(keys))
        t = ctx.timing()
        assert t.passes_possible == 8 and t.passes_executed == 4
        assert np.array_equal(to_host(out, np.int64), oracle.sort(keys))
        u = rand_keys(1 << 18, np.uint32, np.random.default_rng(1))
        ctx.sort(to_dev(u))
        assert ctx.timing().passes_executed == 4
    finally:
        ctx.enable_timing(False)


def test_full_size_cfg2_properties(ctx):
    """cfg2 at full size (2^28 uint32, gen_data stream >> 32): sortedness and the
    multiset hash of input == output, checked on the device."""
    n = 1 << 28
    keys = ctx.gen_keys(n, 1, torch.uint32, shift=32)
    _, _, ms_in = ctx.check_sorted(keys)
    out, _ = ctx.sort(keys)
    inv, _, ms_out = ctx.check_sorted(out)
    assert inv == 0 and ms_in == ms_out
    # a second run is bit-identical (deterministic)
    out2, _ = ctx.sort(keys)
    assert torch.equal(out.view(torch.int32), out2.view(torch.int32))
    # and spot-check a slice against the oracle: the first 2^20 keys sorted
    # alone are a sub-multiset -- compare the global order of a sampled window
    h = to_host(out[: 1 << 16], np.uint32)
    assert np.all(h[1:] >= h[:-1])
    del keys, out, out2
    torch.cuda.empty_cache()


def test_large_pairs_cfg5_shape(ctx):
    """cfg5 shape on one GPU at reduced size: u64 keys (gen_data) + u32 index,
    stable; compared with the oracle's stable merge sort."""
    n = 1 << 22
    keys = ctx.gen_keys(n, 1, torch.uint64, shift=0)
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    ok, ov = ctx.sort(keys, vals=vals)
    torch.cuda.synchronize()
    hk = to_host(keys, np.uint64)
    ek, ev = oracle.stable_sort_kv(hk, np.arange(n, dtype=np.uint32))
    assert np.array_equal(to_host(ok, np.uint64), ek)
    assert np.array_equal(ov.cpu().numpy().view(np.uint32), ev)


def test_device_generator_matches_gen_data(ctx, golden):
    for g in golden["gen_data"]:
        t = ctx.gen_keys(g["n"], g["seed"], torch.int64)
        torch.cuda.synchronize()
        assert oracle.fingerprint(t.cpu().numpy()) == int(g["fp"])
    # windows and shifts of the stream
    full = oracle.gen_data(5000, 3).view(np.uint64)
    t = ctx.gen_keys(1000, 3, torch.int32, shift=33, first=2000)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), (full[2000:3000] >> np.uint64(33)).astype(np.int32))


def test_check_sorted_fingerprint_matches_oracle(ctx):
    rng = np.random.default_rng(2)
    for dt in DTYPES:
        x = rand_keys(10_000, dt, rng)
        inv, fp, _ = ctx.check_sorted(to_dev(x))
        assert fp == oracle.fingerprint(x)
        assert inv == int(np.sum(x[1:] < x[:-1]))


def test_sort_batch_host_pipeline(ctx):
    """b2s_sort_batch: overlapped upload / sort / download of several host arrays."""
    rng = np.random.default_rng(21)
    for dt in DTYPES:
        n = 300_001
        batch = [rand_keys(n, dt, rng, kind) for kind in ("uniform", "dups", "topbyte", "equal", "uniform")]
        outs, _ = ctx.sort_batch(batch)
        for x, o in zip(batch, outs):
            assert np.array_equal(o, oracle.sort(x))
    keys = [rand_keys(100_000, np.uint64, rng, "dups") for _ in range(3)]
    vals = [np.arange(100_000, dtype=np.uint32) for _ in range(3)]
    ok, ov = ctx.sort_batch(keys, vals_list=vals)
    for k, v, a, b in zip(keys, vals, ok, ov):
        ek, ev = oracle.stable_sort_kv(k, v)
        assert np.array_equal(a, ek) and np.array_equal(b, ev)


def test_n_at_least_2p30_uses_64bit_lookback(ctx):
    """n >= 2^30 switches the look-back words to 64 bits (a digit's prefix no
    longer fits 30 bits); sortedness + multiset equality at 2^30 + 12345."""
    n = (1 << 30) + 12345
    keys = ctx.gen_keys(n, 5, torch.int32, shift=32)
    _, _, ms_in = ctx.check_sorted(keys)
    out, _ = ctx.sort(keys)
    inv, _, ms_out = ctx.check_sorted(out)
    assert inv == 0 and ms_in == ms_out
    del keys, out
    torch.cuda.empty_cache()


def test_max_size_cfg3_on_one_gpu(ctx):
    """cfg3 at G=1: all 2^31 int32 keys (z >> 33) sorted on one GPU (64-bit
    look-back words, one prefetched predecessor): sortedness, multiset
    equality with the input and determinism, checked on the device; the
    first key is no larger than the smallest of a 2^24-key input sample."""
    n = 1 << 31
    keys = ctx.gen_keys(n, 1, torch.int32, shift=33)
    _, _, ms_in = ctx.check_sorted(keys)
    out, _ = ctx.sort(keys)
    inv, _, ms_out = ctx.check_sorted(out)
    assert inv == 0 and ms_in == ms_out
    assert int(out[0]) <= int(keys[: 1 << 24].min())
    out2, _ = ctx.sort(keys)
    assert torch.equal(out, out2)
    del keys, out, out2
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("kind", ["uniform", "skewed", "lowzero", "midconst", "topbyte", "sorted",
                                  "extremes", "equal"])
def test_all_digit_prologue_sizes(ctx, dt, kind):
    """From 2^22 keys up, 4-byte keys take every digit histogram from the
    all-digit prologue (signed top digit counted with its sign flip, constant
    digits skipped, no in-pass counting); 8-byte keys the digit-0 prologue
    and in-pass counts (tests/test_gpu_rank_modes.py runs them through the
    8-digit prologue too): bit-exact against numpy."""
    rng = np.random.default_rng(11)
    for n in ((1 << 22) - 1, 1 << 22, (1 << 22) + 12345):
        keys = rand_keys(n, dt, rng, kind)
        out, _ = ctx.sort(to_dev(keys))
        torch.cuda.synchronize()
        assert np.array_equal(to_host(out, dt), np.sort(keys)), (kind, n)


@pytest.mark.parametrize("dt", DTYPES)
def test_all_digit_prologue_pairs_and_unaligned(ctx, dt):
    rng = np.random.default_rng(12)
    n = (1 << 22) + 77
    keys = rand_keys(n, dt, rng, "dups")
    vals = np.arange(n, dtype=np.uint32)
    dv = torch.from_numpy(vals.view(np.int32)).cuda().view(torch.uint32)
    out, vout = ctx.sort(to_dev(keys), vals=dv)
    torch.cuda.synchronize()
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(to_host(out, dt), keys[order])
    assert np.array_equal(vout.view(torch.int32).cpu().numpy().view(np.uint32), order.astype(np.uint32))
    # input one element past a 16-byte boundary: scalar prologue loads, no TMA
    keys = rand_keys(n + 1, dt, rng)
    d = to_dev(keys)[1:]
    out, _ = ctx.sort(d)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out, dt), np.sort(keys[1:]))


def test_lane_ordered_atomics_probe(ctx):
    """On B200 the probe at context creation finds same-word lanes of one
    shared atomic served in lane order -- also with lanes predicated off --
    so the fast ranking is the one in use (a silent fallback to ballot
    matching would stay correct but slow)."""
    assert ctx.lane_ordered_atomics
