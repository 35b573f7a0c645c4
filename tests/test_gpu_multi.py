"""GPU: the multi-GPU sample sort behind the C ABI (b2s_create_multi /
b2s_sample_sort), which stands in for parallel::scatter_merge_sort across
devices (P/src/parallel_sort.cpp:166-254; rank threads as in
runtime::spawn_world, P/src/runtime.cpp:666-694).

On a one-GPU box the ranks are emulated: every rank gets its own context,
stream and host thread on device 0, and the exchange is the p2p pull (a
rank's merge reads its peers' sorted shards; ordering by CUDA events only, so
no kernel waits on another rank). NCCL runs at world size 1 (a communicator
of one device: all-gather and send/recv to itself).

The buckets concatenated in rank order must equal the oracle's sort of the
concatenated shards; with a payload, its stable order (ties by global
index). The full-size cases compare the concatenation with the golden
fingerprints of tests/golden/fullsize.json (cfg3 at G=8, cfg4a-d and cfg5)."""
import json
import os

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1105_6040_b200 import workloads  # noqa: E402
from paper_1105_6040_b200.device import Context, MultiContext  # noqa: E402
from paper_1105_6040_b200.errors import ConfigError, DeviceError  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = {c["config"]: c for c in json.load(open(os.path.join(HERE, "golden", "fullsize.json")))["configs"]}
TORCH = {np.int32: torch.int32, np.uint32: torch.uint32, np.int64: torch.int64, np.uint64: torch.uint64}


def to_dev(x):
    if x.dtype in (np.uint32, np.uint64):
        v = torch.from_numpy(x.view(np.int32 if x.dtype == np.uint32 else np.int64)).cuda()
        return v.view(TORCH[x.dtype.type])
    return torch.from_numpy(x).cuda()


def to_host(t, dt):
    if dt in (np.uint32, np.uint64):
        return t.view(torch.int32 if dt == np.uint32 else torch.int64).cpu().numpy().view(dt)
    return t.cpu().numpy()


def keys_of(kind, n, dt, rng):
    info = np.iinfo(dt)
    if kind == "uniform":
        return rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    if kind == "dups":
        return rng.integers(0, 7, n).astype(dt)
    if kind == "equal":
        return np.full(n, 5, dtype=dt)
    if kind == "sorted":
        return np.sort(rng.integers(info.min, info.max, n, dtype=dt, endpoint=True))
    if kind == "reverse":
        return np.sort(rng.integers(info.min, info.max, n, dtype=dt, endpoint=True))[::-1].copy()
    raise ValueError(kind)


@pytest.fixture(scope="module")
def multis():
    ms = {}
    yield ms
    for m in ms.values():
        m.close()


def multi(multis, G):
    if G not in multis:
        multis[G] = MultiContext([0] * G)
    return multis[G]


def test_info_world1_has_nccl():
    with MultiContext([0]) as m:
        i = m.info()
        assert i["ranks"] == 1 and i["p2p"] and i["nccl"] and i["nccl_version"] >= 22700, i
    with MultiContext([0, 0, 0]) as m:
        i = m.info()
        assert i["ranks"] == 3 and i["p2p"] and not i["nccl"], i  # NCCL refuses one device twice
        with pytest.raises(DeviceError) as e:
            m.set_transport("nccl")
        assert e.value.status == 5  # B2S_ENCCL


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dt", [np.int32, np.uint32, np.int64, np.uint64])
@pytest.mark.parametrize("kind", ["uniform", "dups", "equal", "sorted", "reverse"])
def test_sample_sort_emulated(multis, G, dt, kind):
    rng = np.random.default_rng(G * 131 + np.dtype(dt).itemsize + len(kind))
    n = 300_001
    data = keys_of(kind, n, dt, rng)
    sizes = oracle.plan_partition(n, G)
    shards, off = [], 0
    for s in sizes:
        shards.append(data[off: off + s].copy())
        off += s
    m = multi(multis, G)
    buckets, _ = m.sample_sort([to_dev(x) for x in shards])
    got = np.concatenate([to_host(b, dt) for b in buckets])
    assert np.array_equal(got, oracle.sort(data))
    t = m.timing()
    assert t.transport == "p2p"
    assert t.max_bucket <= 2 * (n // G) + 64 * G + 1024, (t.max_bucket, n, G)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("dt", [np.int32, np.uint64])
@pytest.mark.parametrize("kind", ["dups", "equal", "uniform"])
def test_sample_sort_pairs_stable(multis, G, dt, kind):
    """Payload = global index: the concatenated payloads must be the stable
    order (ties by shard order, then position)."""
    rng = np.random.default_rng(7 * G + len(kind))
    n = 200_003
    data = keys_of(kind, n, dt, rng)
    idx = np.arange(n, dtype=np.uint32)
    ek, ev = oracle.stable_sort_kv(data, idx)
    sizes = oracle.plan_partition(n, G)
    shards, vals, off = [], [], 0
    for s in sizes:
        shards.append(to_dev(data[off: off + s].copy()))
        vals.append(to_dev(idx[off: off + s].copy()))
        off += s
    m = multi(multis, G)
    buckets, bvals = m.sample_sort(shards, vals=vals)
    gk = np.concatenate([to_host(b, dt) for b in buckets])
    gv = np.concatenate([to_host(b, np.uint32) for b in bvals])
    assert np.array_equal(gk, ek) and np.array_equal(gv, ev)


def test_empty_and_ragged_shards(multis):
    rng = np.random.default_rng(3)
    shards = [np.zeros(0, np.int32), rng.integers(-50, 50, 1000).astype(np.int32),
              np.zeros(0, np.int32), rng.integers(-50, 50, 7).astype(np.int32)]
    m = multi(multis, 4)
    buckets, _ = m.sample_sort([to_dev(x) if x.size else torch.empty(0, dtype=torch.int32, device="cuda")
                                for x in shards])
    got = np.concatenate([b.cpu().numpy() for b in buckets])
    assert np.array_equal(got, np.sort(np.concatenate(shards)))
    # all empty
    buckets, _ = m.sample_sort([torch.empty(0, dtype=torch.int32, device="cuda")] * 4)
    assert sum(b.numel() for b in buckets) == 0


def test_host_buffers(multis):
    rng = np.random.default_rng(5)
    shards = [rng.integers(0, 2**63, 50_000, dtype=np.int64) for _ in range(3)]
    vals = [np.arange(i * 50_000, (i + 1) * 50_000, dtype=np.uint32) for i in range(3)]
    m = multi(multis, 3)
    buckets, bvals = m.sample_sort(shards, vals=vals)  # numpy: B2S_HOST
    allk = np.concatenate(shards)
    ek, ev = oracle.stable_sort_kv(allk, np.arange(allk.size, dtype=np.uint32))
    assert np.array_equal(np.concatenate(buckets), ek)
    assert np.array_equal(np.concatenate(bvals), ev)


def test_nccl_transport_world1():
    """NCCL at world size 1: the all-gathers and the grouped send/recv run
    through a real communicator (the only NCCL a one-GPU box can run)."""
    rng = np.random.default_rng(11)
    data = rng.integers(-2**31, 2**31 - 1, 1 << 20, dtype=np.int64).astype(np.int32)
    idx = np.arange(data.size, dtype=np.uint32)
    with MultiContext([0]) as m:
        m.set_transport("nccl")
        buckets, bvals = m.sample_sort([to_dev(data)], vals=[to_dev(idx)])
        assert m.timing().transport == "nccl"
        ek, ev = oracle.stable_sort_kv(data, idx)
        assert np.array_equal(buckets[0].cpu().numpy(), ek)
        assert np.array_equal(to_host(bvals[0], np.uint32), ev)


def test_capacity_error(multis):
    m = multi(multis, 2)
    x = torch.arange(1000, dtype=torch.int32, device="cuda")
    outs = [torch.empty(10, dtype=torch.int32, device="cuda") for _ in range(2)]
    with pytest.raises(ConfigError):
        m.sample_sort([x, x.clone()], outs=outs, capacity=[10, 10])


# ---- full size (BASELINE configs), emulated G=8 on one GPU ------------------

def _concat_fp(buckets, vals=None):
    ctx = Context(0)
    try:
        cat = torch.cat(buckets)
        inv, fp, ms = ctx.check_sorted(cat)
        vfp = None
        if vals is not None:
            _, vfp, _ = ctx.check_sorted(torch.cat(vals))
        return inv, fp, ms, vfp, cat.numel()
    finally:
        ctx.close()


def _shards(gen, total, G):
    sizes = oracle.plan_partition(total, G)
    out, off = [], 0
    for s in sizes:
        out.append(gen(s, off))
        off += s
    return out


def test_cfg3_g8_full(multis):
    G, N = 8, 1 << 31
    ctx = Context(0)
    shards = _shards(lambda s, off: ctx.gen_keys(s, 1, torch.int32, shift=33, first=off), N, G)
    ctx.close()
    m = multi(multis, G)
    buckets, _ = m.sample_sort(shards)
    del shards
    inv, fp, ms, _, n = _concat_fp(buckets)
    g = GOLD["cfg3"]
    assert n == N and inv == 0 and ms == int(g["multiset"]) and fp == int(g["fp"])
    t = m.timing()
    assert t.max_bucket <= 2 * N // G
    del buckets
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kind,name", [("zipf", "cfg4a"), ("ascending", "cfg4b"),
                                       ("descending", "cfg4c"), ("equal", "cfg4d")])
def test_cfg4_g8_full(multis, kind, name):
    G, N = 8, 1 << 27
    ctx = Context(0)
    shards = _shards(lambda s, off: workloads.cfg4_keys(ctx, kind, s, first=off, total=N), N, G)
    ctx.close()
    m = multi(multis, G)
    buckets, _ = m.sample_sort(shards)
    inv, fp, ms, _, n = _concat_fp(buckets)
    g = GOLD[name]
    assert n == N and inv == 0 and ms == int(g["multiset"]) and fp == int(g["fp"]), name
    # compound samples keep skewed / all-equal buckets balanced
    assert m.timing().max_bucket <= 2 * N // G, (name, m.timing())


def test_cfg5_g8_full(multis):
    G, N = 8, 1 << 28
    ctx = Context(0)
    shards = _shards(lambda s, off: ctx.gen_keys(s, 1, torch.uint64, first=off), N, G)
    vals = _shards(lambda s, off: torch.arange(off, off + s, dtype=torch.int64, device="cuda")
                   .to(torch.int32).view(torch.uint32), N, G)
    ctx.close()
    m = multi(multis, G)
    buckets, bvals = m.sample_sort(shards, vals=vals)
    inv, fp, ms, vfp, n = _concat_fp(buckets, bvals)
    g = GOLD["cfg5"]
    assert n == N and inv == 0 and ms == int(g["multiset"]) and fp == int(g["fp"])
    assert vfp == int(g["payload_fp"])


def test_run_benchmark_multi_exp1_row():
    """bench::run_benchmark / exp1 row (P/src/bench.cpp:106-169,211-222) with
    procs = GPU ranks of the sample sort, verified every repetition."""
    from paper_1105_6040_b200 import report as R
    for m in (1, 2, 4):
        rep = R.run_benchmark_multi(R.RunConfig("merge", 1 << 18, m, 2, 1, "wall", 2), [0] * m)
        row = R.exp1_csv_row(rep).split(",")
        assert row[0] == "merge" and row[2] == str(m) and float(row[4]) > 0
        kinds = {e.kind for e in rep.world.trace}
        assert kinds == {"compute", "bcast", "gather"} and len(rep.world.trace) == 3 * m
