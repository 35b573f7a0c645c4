"""GPU: the upper-digits-first path of 8-byte keys (radix_sort.cu,
radix_plan_kernel / topfirst_fixup_kernel). From 2^22 to 2^31 keys whose upper
halves vary in enough bits, only the four upper digits are radix-sorted and a
fix-up kernel orders the few ties by their lower halves; inputs the fix-up
cannot finish (long tie runs) fall back to a full second sort. Every case is
compared bit-exactly with numpy's stable sort (the reference's merge_sort tie
rule, P/src/sort_core.cpp:77), keys and payload, and the pass counters say
which path ran."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1105_6040_b200.device import Context  # noqa: E402

N = (1 << 22) + 12345  # ragged last tile, just inside the path's size window


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    c.enable_timing(True)
    yield c
    c.close()


def to_dev(x):
    if x.dtype == np.uint64:
        return torch.from_numpy(x.view(np.int64)).cuda().view(torch.uint64)
    if x.dtype == np.uint32:
        return torch.from_numpy(x.view(np.int32)).cuda().view(torch.uint32)
    return torch.from_numpy(x).cuda()


def to_host(t, dt):
    if dt == np.uint64:
        return t.view(torch.int64).cpu().numpy().view(np.uint64)
    if dt == np.uint32:
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.cpu().numpy()


def check(ctx, keys, passes, with_vals=True):
    """Sorts keys (and an index payload) on the device; compares with numpy's
    stable sort; returns after asserting the executed pass count."""
    order = np.argsort(keys, kind="stable")
    out, _ = ctx.sort(to_dev(keys))
    t = ctx.timing()
    assert np.array_equal(to_host(out, keys.dtype.type), keys[order])
    if passes is not None:
        assert t.passes_executed == passes, t
    if with_vals:
        vals = np.arange(keys.size, dtype=np.uint32)
        ok, ov = ctx.sort(to_dev(keys), vals=to_dev(vals))
        assert np.array_equal(to_host(ok, keys.dtype.type), keys[order])
        assert np.array_equal(to_host(ov, np.uint32), order.astype(np.uint32))
        # in place, keys and payload
        k2, v2 = to_dev(keys), to_dev(vals)
        ctx.sort(k2, out=k2, vals=v2, vals_out=v2)
        assert np.array_equal(to_host(k2, keys.dtype.type), keys[order])
        assert np.array_equal(to_host(v2, np.uint32), order.astype(np.uint32))


@pytest.mark.parametrize("dt", [np.uint64, np.int64])
def test_uniform_runs_four_passes(ctx, dt):
    rng = np.random.default_rng(7)
    info = np.iinfo(dt)
    keys = rng.integers(info.min, info.max, N, dtype=dt, endpoint=True)
    check(ctx, keys, 4)


def test_ties_of_the_upper_half_are_ordered_by_the_fixup(ctx):
    """~8 keys per upper half, random lower halves: every run needs the
    insertion sort, none is too long; the payload shows the order is stable."""
    rng = np.random.default_rng(8)
    tops = rng.integers(0, 1 << 32, N // 8, dtype=np.uint64)
    hi = tops[rng.integers(0, tops.size, N)]
    lo = rng.integers(0, 1 << 8, N, dtype=np.uint64)  # few lower values: full-key duplicates too
    keys = (hi << np.uint64(32)) | lo
    check(ctx, keys, 4)


def test_long_unsorted_runs_fall_back_to_the_full_sort(ctx):
    """512 distinct upper halves (digit 4 looks spread out), random lower
    halves: runs of ~8000 unsorted keys, so the fix-up raises its flag."""
    rng = np.random.default_rng(9)
    tops = rng.integers(0, 1 << 32, 512, dtype=np.uint64)
    hi = tops[rng.integers(0, tops.size, N)]
    lo = rng.integers(0, 1 << 32, N, dtype=np.uint64)
    keys = (hi << np.uint64(32)) | lo
    check(ctx, keys, 4)  # the first sort's counters are the reported ones


def test_few_distinct_upper_halves_take_the_plain_path(ctx):
    """Four upper halves that differ in every bit: digit 4 is concentrated,
    so the plan does not try the upper digits first."""
    rng = np.random.default_rng(17)
    tops = np.array([0x00000000, 0xFFFFFFFF, 0x5A5A5A5A, 0xA5A5A5A5], dtype=np.uint64)
    hi = tops[rng.integers(0, 4, N)]
    lo = rng.integers(0, 1 << 32, N, dtype=np.uint64)
    check(ctx, (hi << np.uint64(32)) | lo, 8)


def test_long_sorted_runs_fall_back(ctx):
    """Runs longer than the fix-up's scan window, already in order (equal
    keys): flagged, and the full sort keeps the payload stable."""
    rng = np.random.default_rng(10)
    tops = rng.integers(0, 1 << 32, 512, dtype=np.uint64)
    hi = tops[rng.integers(0, tops.size, N)]
    keys = (hi << np.uint64(32)) | np.uint64(12345)
    check(ctx, keys, 4)


def test_runs_just_past_the_insertion_limit(ctx):
    """Unsorted runs of 33..40 keys (limit 32) among short ones."""
    rng = np.random.default_rng(11)
    n_long = 1000
    long_tops = rng.integers(0, 1 << 32, n_long, dtype=np.uint64)
    reps = rng.integers(33, 41, n_long)
    hi_long = np.repeat(long_tops, reps)
    rest = N - hi_long.size
    hi = np.concatenate([hi_long, rng.integers(0, 1 << 32, rest, dtype=np.uint64)])
    rng.shuffle(hi)
    lo = rng.integers(0, 1 << 32, N, dtype=np.uint64)
    check(ctx, (hi << np.uint64(32)) | lo, 4)


def test_runs_at_the_insertion_limit_stay_on_the_fixup(ctx):
    """Runs of exactly 32: the longest the fix-up sorts itself."""
    rng = np.random.default_rng(12)
    tops = rng.integers(0, 1 << 32, N // 32 + 1, dtype=np.uint64)
    hi = np.repeat(tops, 32)[:N].copy()
    rng.shuffle(hi)
    lo = rng.integers(0, 1 << 32, N, dtype=np.uint64)
    check(ctx, (hi << np.uint64(32)) | lo, 4, with_vals=False)


def test_narrow_upper_half_takes_the_plain_path(ctx):
    """Keys below 2^40: 8 varying upper bits are too few, all 5 digits run."""
    rng = np.random.default_rng(13)
    keys = rng.integers(0, 1 << 40, N, dtype=np.uint64)
    check(ctx, keys, 5)


def test_constant_lower_half_takes_the_plain_path(ctx):
    rng = np.random.default_rng(14)
    keys = rng.integers(0, 1 << 32, N, dtype=np.uint64) << np.uint64(32)
    check(ctx, keys, 4, with_vals=False)


def test_run_at_the_array_ends(ctx):
    """Tie runs touching the first and the last element."""
    rng = np.random.default_rng(15)
    keys = rng.integers(0, 1 << 64, N, dtype=np.uint64)
    srt = np.sort(keys)
    lo3 = np.array([3, 1, 2], dtype=np.uint64)
    keys[:3] = (srt[0] & ~np.uint64(0xFFFFFFFF)) | lo3          # smallest upper half
    keys[-3:] = (srt[-1] | np.uint64(0xFFFFFFFF)) - lo3          # largest upper half
    check(ctx, keys, 4)


def test_below_the_window_runs_all_passes(ctx):
    rng = np.random.default_rng(16)
    keys = rng.integers(0, 1 << 64, (1 << 22) - 1, dtype=np.uint64)
    check(ctx, keys, 8, with_vals=False)


def test_two_to_the_thirty_keys(ctx):
    """2^30 uniform uint64 keys: a quarter of the upper-half classes are
    shared, so the fix-up handles ~22% of the keys; compared with torch.sort
    (order-preserving signed view)."""
    n = 1 << 30
    keys = ctx.gen_keys(n, 5, torch.uint64, shift=0)
    out, _ = ctx.sort(keys)
    assert ctx.timing().passes_executed == 4
    ref = torch.sort(keys.view(torch.int64) ^ torch.iinfo(torch.int64).min)[0]
    del keys
    assert torch.equal(out.view(torch.int64) ^ torch.iinfo(torch.int64).min, ref)
    del out, ref
    torch.cuda.empty_cache()
