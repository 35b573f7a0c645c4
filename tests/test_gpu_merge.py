"""GPU: merge-path merges (b2s_merge, b2s_merge_split_padded) and the
single-GPU partitioned sort against the oracle, including kernels::merge_runs'
tie rule (ties from the lower run) checked through a payload."""
import os

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1105_6040_b200.device import Context  # noqa: E402
from test_gpu_sort import DTYPES, rand_keys, to_dev, to_host  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 7, 8, 9, 16])
def test_kway_merge(ctx, dt, k):
    _kway_case(ctx, dt, k)


@pytest.mark.parametrize("mode,k", [("1", 3), ("1", 8), ("1", 16), ("0", 3), ("0", 8)])
def test_kway_merge_modes(mode, k):
    """Both k-way strategies whatever the default picks: the grouped
    single-pass merge forced on (B2S_KWAY=1, also for 8-byte keys and k > 8)
    and the pairwise rounds forced on (B2S_KWAY=0), each in a subprocess so
    the mode switch is read fresh."""
    import subprocess
    import sys
    code = ("import sys; sys.path[:0] = [%r, %r]\n"
            "import numpy as np, test_gpu_merge as t\n"
            "from paper_1105_6040_b200.device import Context\n"
            "c = Context(0)\n"
            "for dt in t.DTYPES: t._kway_case(c, dt, %d)\n"
            "print('ok')") % (os.path.dirname(__file__), os.path.dirname(os.path.dirname(__file__)), k)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, B2S_KWAY=mode),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def _kway_case(ctx, dt, k):
    rng = np.random.default_rng(k * 31 + np.dtype(dt).itemsize)
    for kind in ("uniform", "dups"):
        lens = [int(x) for x in rng.integers(0, 20_000, k)]
        if k > 2:
            lens[1] = 0  # an empty run in the middle
        runs = [oracle.sort(rand_keys(n, dt, rng, kind)) for n in lens]
        out, _ = ctx.merge([to_dev(r) for r in runs])
        torch.cuda.synchronize()
        assert np.array_equal(to_host(out, dt), oracle.merge_kway(runs)), (kind, lens)
        hout, _ = ctx.merge(runs)  # host buffers
        assert np.array_equal(hout, oracle.merge_kway(runs))


@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_kway_merge_ties_take_lower_run(ctx, k):
    """Stability: equal keys come out in run order, then position order
    (merge_runs' rule, P/src/sort_core.cpp:46, tested at
    P/tests/test_sort_core.cpp:110-120)."""
    rng = np.random.default_rng(k)
    runs, vals, off = [], [], 0
    for _ in range(k):
        n = int(rng.integers(1000, 30_000))
        runs.append(np.sort(rng.integers(0, 8, n).astype(np.uint32)))
        vals.append(np.arange(off, off + n, dtype=np.uint32))
        off += n
    ek, ev = oracle.stable_sort_kv(np.concatenate(runs), np.concatenate(vals))
    ok, ov = ctx.merge([to_dev(r) for r in runs],
                       vals=[torch.from_numpy(v.view(np.int32)).cuda() for v in vals])
    torch.cuda.synchronize()
    assert np.array_equal(to_host(ok, np.uint32), ek)
    assert np.array_equal(ov.cpu().numpy().view(np.uint32), ev)


def test_merge_runs_kats(ctx, golden):
    for m in golden["merge_runs"]:
        a = np.array(m["a"], dtype=np.int64)
        b = np.array(m["b"], dtype=np.int64)
        out, _ = ctx.merge([a, b])
        assert out.tolist() == m["expected"]


def test_merge_rejects_aliasing_output(ctx):
    from paper_1105_6040_b200.errors import ConfigError
    x = torch.arange(100, dtype=torch.int64, device="cuda")
    with pytest.raises(ConfigError):
        ctx.merge([x[:50], x[50:]], out=x)


def test_merge_split_padded_golden(ctx, golden):
    for c in golden["merge_split_padded"]:
        reals, virt = ctx.merge_split_padded(np.array(c["mine"], dtype=np.int64),
                                             c["mine_virt"],
                                             np.array(c["theirs"], dtype=np.int64),
                                             c["theirs_virt"], c["keep"] == "high")
        assert reals.tolist() == c["reals"] and virt == c["virtuals"], c


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8, 13, 64])
def test_partitioned_sort(ctx, dt, p):
    rng = np.random.default_rng(p)
    for n in (0, 5, 4097, 250_001):
        keys = rand_keys(n, dt, rng, "uniform" if n % 2 else "dups")
        out, _ = ctx.partitioned_sort(to_dev(keys), p)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(out, dt), oracle.sort(keys)), (n, p)


def test_partitioned_sort_pairs_stable(ctx):
    rng = np.random.default_rng(4)
    n = 300_000
    keys = rng.integers(0, 100, n).astype(np.int64)
    vals = np.arange(n, dtype=np.uint32)
    ek, ev = oracle.stable_sort_kv(keys, vals)
    for p in (1, 3, 4, 8):
        ok, ov = ctx.partitioned_sort(keys, p, vals=vals)
        assert np.array_equal(ok, ek) and np.array_equal(ov, ev), p


def test_merge_empty_runs_with_payload(ctx):
    """Regression: an empty run carries a null payload pointer; the payload of
    the other runs must still be merged."""
    k = torch.full((5000,), 7, dtype=torch.int32, device="cuda")
    v = torch.arange(5000, dtype=torch.int32, device="cuda")
    e, ev = k[:0], v[:0]
    for runs, vals in (([e, k], [ev, v]), ([k, e], [v, ev]), ([e, k, e, k], [ev, v, ev, v])):
        ok, ov = ctx.merge(runs, vals=vals)
        torch.cuda.synchronize()
        assert torch.equal(ov, torch.cat([x for x in vals]))


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_repeated_calls_see_new_data(ctx, dt):
    """Repeated device calls on the same buffers (partitioned, out-of-place and
    in-place sorts) sort the buffers' current contents, also after a larger
    call reallocated the context's scratch."""
    rng = np.random.default_rng(11)
    n, p = 300_001, 4
    d_in = to_dev(rand_keys(n, dt, rng))
    d_out = torch.empty_like(d_in)
    for it in range(6):
        keys = rand_keys(n, dt, rng, "uniform" if it % 2 else "dups")
        d_in.copy_(to_dev(keys))
        ctx.partitioned_sort(d_in, p, out=d_out)
        s_out, _ = ctx.sort(d_in)  # fresh output each time
        ctx.sort(d_in, out=d_in)   # in place, same pointers
        torch.cuda.synchronize()
        expect = oracle.sort(keys)
        assert np.array_equal(to_host(d_out, dt), expect), it
        assert np.array_equal(to_host(d_in, dt), expect), it
        assert np.array_equal(to_host(s_out, dt), expect), it
        if it == 3:  # grow every scratch buffer
            big = to_dev(rand_keys(3 * n, dt, rng))
            ctx.partitioned_sort(big, p)


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_partitioned_sort_graph_replay(ctx, dt):
    """Small partitioned sorts replay a captured CUDA graph from the second
    identical call on: every call sorts the buffers' current contents, a
    replay launches the captured kernels (counted), and a call of another
    shape or after scratch reallocation takes the direct path again."""
    from paper_1105_6040_b200._lib import lib
    rng = np.random.default_rng(21)
    n, p = 1 << 20, 4
    d_in = to_dev(rand_keys(n, dt, rng))
    d_out = torch.empty_like(d_in)
    counts = []
    for it in range(6):
        keys = rand_keys(n, dt, rng, ("uniform", "dups", "sorted", "skewed", "equal", "reverse")[it])
        d_in.copy_(to_dev(keys))
        l0 = lib().b2s_kernel_launches()
        ctx.partitioned_sort(d_in, p, out=d_out)
        counts.append(lib().b2s_kernel_launches() - l0)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(d_out, dt), oracle.sort(keys)), it
        if it == 3:  # another shape, then a scratch reallocation, in between
            other = to_dev(rand_keys(n // 2, dt, rng))
            o2, _ = ctx.partitioned_sort(other, 3)
            big = to_dev(rand_keys(4 * n, dt, rng))
            ctx.partitioned_sort(big, p)
            torch.cuda.synchronize()
            assert np.array_equal(to_host(o2, dt), oracle.sort(to_host(other, dt)))
    assert all(c > 0 for c in counts), counts
    assert counts[2] == counts[3] == counts[0], counts  # replays count the captured kernels


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8, 13])
def test_odd_even_sort(ctx, dt, p):
    """The reference's own p-phase algorithm on the device (radix-sorted
    blocks, p odd-even merge_split_padded phases, rank-order gather):
    bit-exact with the oracle's restatement of scatter_merge_sort (int64) and
    with the sorted input (other key types)."""
    rng = np.random.default_rng(100 + p)
    for n in (0, 5, 4097, 250_001):
        keys = rand_keys(n, dt, rng, "uniform" if n % 2 else "dups")
        out = ctx.odd_even_sort(to_dev(keys), p)
        torch.cuda.synchronize()
        if dt == np.int64:
            expect = oracle.scatter_merge_sort(keys, p)
        else:
            expect = np.sort(keys)
        assert np.array_equal(to_host(out, dt), expect), (n, p)
    # host buffers
    keys = rand_keys(10_000, dt, rng)
    assert np.array_equal(ctx.odd_even_sort(keys, p), np.sort(keys))
