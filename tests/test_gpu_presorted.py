"""GPU: presorted input (radix_sort.cu, radix_order_check_kernel). From 2^20 keys
on, when the prologue's sample of adjacent pairs is all one way, every
adjacent pair is counted: ascending input runs no pass (cfg4b), descending
input is reversed (cfg4c) -- with a payload only when strictly decreasing, so
equal keys keep their input order (merge_sort's tie rule,
P/src/sort_core.cpp:77). One inversion anywhere must send the sort down the
regular passes. Results are compared bit-exactly with numpy's stable sort."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1105_6040_b200.device import Context  # noqa: E402

DTYPES = [np.int32, np.uint32, np.int64, np.uint64]
TORCH = {np.int32: torch.int32, np.uint32: torch.uint32, np.int64: torch.int64,
         np.uint64: torch.uint64}
N = (1 << 20) + 37  # not a whole number of 16-byte vectors


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    c.enable_timing(True)
    yield c
    c.close()


def to_dev(x):
    if x.dtype in (np.uint32, np.uint64):
        wire = np.int32 if x.dtype == np.uint32 else np.int64
        return torch.from_numpy(x.view(wire)).cuda().view(TORCH[x.dtype.type])
    return torch.from_numpy(x).cuda()


def to_host(t, dt):
    if dt in (np.uint32, np.uint64):
        return t.view(torch.int32 if dt == np.uint32 else torch.int64).cpu().numpy().view(dt)
    return t.cpu().numpy()


def run(ctx, keys, vals=None, in_place=False):
    dk = to_dev(keys)
    dv = to_dev(vals) if vals is not None else None
    if in_place:
        ok, ov = ctx.sort(dk, out=dk, vals=dv, vals_out=dv)
    else:
        ok, ov = ctx.sort(dk, vals=dv)
    t = ctx.timing()
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(to_host(ok, keys.dtype.type), keys[order])
    if vals is not None:
        assert np.array_equal(to_host(ov, np.uint32), vals[order])
    return t.passes_executed


def sorted_keys(dt, n, rng, strict=False):
    info = np.iinfo(dt)
    if strict:  # distinct values spanning the sign boundary of signed types
        step = (int(info.max) - int(info.min)) // (n + 1)
        return (int(info.min) + step * np.arange(1, n + 1, dtype=object)).astype(dt)
    return np.sort(rng.integers(info.min, info.max, n, dtype=dt, endpoint=True))


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("in_place", [False, True])
def test_ascending_runs_no_pass(ctx, dt, in_place):
    rng = np.random.default_rng(1)
    keys = sorted_keys(dt, N, rng)
    keys[1000:1100] = keys[1000]  # duplicates
    assert run(ctx, keys, in_place=in_place) == 0
    vals = rng.integers(0, 1 << 32, N, dtype=np.uint32)
    assert run(ctx, keys, vals, in_place=in_place) == 0


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("in_place", [False, True])
@pytest.mark.parametrize("n", [N, 1 << 20, (1 << 20) + 2])
def test_strictly_descending_is_reversed(ctx, dt, in_place, n):
    rng = np.random.default_rng(2)
    keys = sorted_keys(dt, n, rng, strict=True)[::-1].copy()
    assert run(ctx, keys, in_place=in_place) == 0
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint32)
    assert run(ctx, keys, vals, in_place=in_place) == 0


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_descending_with_duplicates(ctx, dt):
    """Keys only: reversed. With a payload the reversal would swap equal keys,
    so the regular passes run."""
    rng = np.random.default_rng(3)
    keys = sorted_keys(dt, N, rng)[::-1].copy()
    keys[5000:5003] = keys[5000]
    assert run(ctx, keys) == 0
    vals = np.arange(N, dtype=np.uint32)
    assert run(ctx, keys, vals) > 0


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("pos", [0, 3, 4, 127, 128, 12287, 12288, N - 2])
def test_one_inversion_takes_the_regular_passes(ctx, dt, pos):
    """A single out-of-order pair -- at the first pair, inside a 16-byte
    vector, across vectors, across warps and tiles, at the last pair."""
    rng = np.random.default_rng(4)
    keys = sorted_keys(dt, N, rng, strict=True)
    keys[pos], keys[pos + 1] = keys[pos + 1], keys[pos]
    assert run(ctx, keys) > 0
    desc = sorted_keys(dt, N, rng, strict=True)[::-1].copy()
    desc[pos], desc[pos + 1] = desc[pos + 1], desc[pos]
    assert run(ctx, desc) > 0


@pytest.mark.parametrize("dt", [np.uint32, np.int64])
def test_unaligned_views(ctx, dt):
    """Input and output views one element off a 16-byte boundary."""
    rng = np.random.default_rng(5)
    keys = sorted_keys(dt, N, rng, strict=True)
    for arr in (keys, keys[::-1].copy()):
        big = to_dev(np.concatenate([arr[:1], arr]))
        src = big[1:]
        out = torch.empty(N + 1, dtype=src.dtype, device="cuda")[1:]
        ctx.sort(src, out=out)
        assert ctx.timing().passes_executed == 0
        assert np.array_equal(to_host(out, dt), np.sort(arr))
        ctx.sort(src, out=src)  # in place, unaligned
        assert np.array_equal(to_host(src, dt), np.sort(arr))


def test_random_input_is_not_checked(ctx):
    rng = np.random.default_rng(6)
    keys = rng.integers(0, 1 << 32, N, dtype=np.uint32)
    assert run(ctx, keys) == 4
