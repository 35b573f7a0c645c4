"""GPU: the reference's own result-pinning tests, restated against the B200
path through the reference-shaped API (paper_1105_6040_b200.sortbench) and the
golden fixtures produced by the reference library (tests/golden)."""
import os

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1105_6040_b200 import sortbench as sb  # noqa: E402
from paper_1105_6040_b200.device import default_context  # noqa: E402
from paper_1105_6040_b200.errors import ConfigError, ProgrammingError, VerificationError  # noqa: E402


def opts(p):
    return sb.WorldOptions(procs=p)


def test_acceptance_criterion_1(golden):
    """P/tests/acceptance.cpp:121-157: 1000 seeded cases, n in [0, 4096],
    p in {1,2,3,4,8}, all three algorithms; output == reference output."""
    for c in golden["acceptance1"]:
        data = sb.gen_data(c["n"], int(c["seed"]))
        out = sb.scatter_merge_sort(sb.Algorithm[c["algo"]], data, opts(c["p"])).sorted
        assert oracle.fingerprint(out) == int(c["fp"]), c


def test_random_oracle_equivalence(golden):
    """P/tests/test_parallel_sort.cpp:330-343."""
    for c in golden["random_oracle"]:
        data = sb.gen_data(c["n"], int(c["seed"]))
        out = sb.scatter_merge_sort(sb.Algorithm[c["algo"]], data, opts(c["p"])).sorted
        assert oracle.fingerprint(out) == int(c["fp"])


def test_kats(golden):
    for k in golden["kats"]:
        out = sb.scatter_merge_sort(sb.Algorithm[k["algo"]], np.array(k["input"], dtype=np.int64),
                                    opts(k["p"])).sorted
        assert np.asarray(out).tolist() == k["expected"], k["name"]


def test_quick_p4_gen_data_4096():
    """P/tests/test_parallel_sort.cpp:307-312."""
    data = sb.gen_data(4096, 2024)
    out = sb.scatter_merge_sort(sb.Algorithm.quick, data, opts(4)).sorted
    assert np.array_equal(out, oracle.sort(data))


def test_exhaustive_01():
    """P/tests/test_parallel_sort.cpp:314-328 (n <= 8) and acceptance
    criterion 2 exactly (P/tests/acceptance.cpp:160-189): every 0/1 input of
    n <= 12 keys at p in {2, 3, 4}, 24,573 sorts."""
    for p in (2, 3, 4):
        for n in range(13):
            for mask in range(1 << n):
                data = np.array([(mask >> i) & 1 for i in range(n)], dtype=np.int64)
                out = sb.scatter_merge_sort(sb.Algorithm.bubble, data, opts(p)).sorted
                assert np.asarray(out).tolist() == sorted(data.tolist()), (p, n, mask)


def test_kernel_oracle_stream(golden):
    """P/tests/test_sort_core.cpp:191-216: every local kernel through KernelFn."""
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "kernel_oracle.npz"))
    sizes, values = z["sizes"], z["values"].astype(np.int64)
    off = 0
    for s, fp in zip(sizes, golden["kernel_oracle_merge_fp"]):
        s = int(s)
        for algo in sb.Algorithm:
            blk = values[off: off + s].copy()
            sb.select_kernel(algo)(blk, None)
            assert oracle.fingerprint(blk) == int(fp)
        blk = values[off: off + s].copy()
        sb.merge_sort(blk, 0, s - 1)
        assert oracle.fingerprint(blk) == int(fp)
        off += s


def test_kernel_edge_semantics():
    # merge_sort: first > last is an empty no-op (P/tests/test_sort_core.cpp:144-151)
    v = np.array([3, 1], dtype=np.int64)
    sb.merge_sort(v, 1, 0)
    assert v.tolist() == [3, 1]
    # quick_sort: length <= 1 untouched; out-of-range -> ProgrammingError (:156-183)
    v = np.array([2, 1], dtype=np.int64)
    sb.quick_sort(v, 0, 1)
    assert v.tolist() == [2, 1]
    with pytest.raises(ProgrammingError):
        sb.quick_sort(np.array([1, 2], dtype=np.int64), 1, 2)
    # size_t arguments in the reference: negative values are out of range, not
    # Python's wrap-around slices
    for start, length in ((-1, 1), (0, -1), (-2, 2)):
        with pytest.raises(ProgrammingError):
            sb.quick_sort(np.array([3, 2, 1], dtype=np.int64), start, length)
    # sub-range sorts leave the rest alone
    v = np.array([9, 5, 3, 1, 0], dtype=np.int64)
    sb.merge_sort(v, 1, 3)
    assert v.tolist() == [9, 1, 3, 5, 0]
    assert sb.is_sorted([]) and sb.is_sorted([1, 2, 2, 3]) and not sb.is_sorted([2, 1])
    with pytest.raises(ConfigError):
        sb.scatter_merge_sort(sb.Algorithm.merge, np.arange(4), opts(0))


def test_merge_runs_and_merge_split(golden):
    for m in golden["merge_runs"]:
        assert np.asarray(sb.merge_runs(m["a"], m["b"])).tolist() == m["expected"]
    # P/tests/test_parallel_sort.cpp:125-135
    assert sb.merge_split([1, 3, 5], [2, 4, 6], sb.KeepHalf.low).tolist() == [1, 2, 3]
    assert sb.merge_split([2, 4, 6], [1, 3, 5], sb.KeepHalf.high).tolist() == [4, 5, 6]
    assert sb.merge_split([1, 2], [0, 0, 0], sb.KeepHalf.low).tolist() == [0, 0]
    assert sb.merge_split([], [1], sb.KeepHalf.low).tolist() == []
    for c in golden["merge_split_padded"]:
        r = sb.merge_split_padded(sb.PaddedBlock(np.array(c["mine"], dtype=np.int64),
                                                 c["mine_virt"]),
                                  sb.PaddedBlock(np.array(c["theirs"], dtype=np.int64),
                                                 c["theirs_virt"]),
                                  sb.KeepHalf[c["keep"]])
        assert r.reals.tolist() == c["reals"] and r.virtuals == c["virtuals"]


def test_merge_split_random_oracle():
    """P/tests/test_parallel_sort.cpp:138-169 restated with numpy seeds."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        a = np.sort(rng.integers(0, 8, int(rng.integers(0, 20)))).astype(np.int64)
        b = np.sort(rng.integers(0, 8, int(rng.integers(0, 20)))).astype(np.int64)
        low = sb.merge_split(a, b, sb.KeepHalf.low)
        high = sb.merge_split(b, a, sb.KeepHalf.high)
        assert np.array_equal(low, oracle.merge_split(a, b, False))
        assert np.array_equal(high, oracle.merge_split(b, a, True))


def test_config_pins(golden):
    """cfg1-shaped inputs at full size (N=2^20 int32 = z>>33, p=4, and
    variants), generated on the device; fingerprint == reference output's."""
    ctx = default_context(0)
    for c in golden["config_pins"]:
        if c["shift"]:
            keys = ctx.gen_keys(c["n"], c["seed"], torch.int32, shift=c["shift"])
        else:
            keys = ctx.gen_keys(c["n"], c["seed"], torch.int64)
        out, _ = ctx.partitioned_sort(keys, c["p"])
        inv, fp, _ = ctx.check_sorted(out)
        assert inv == 0 and fp == int(c["fp"]), c


def test_verify_output():
    """P/tests/test_bench.cpp:73-84."""
    inp = np.array([3, 1, 2, 2], dtype=np.int64)
    sb.verify_output(inp, np.array([1, 2, 2, 3], dtype=np.int64))
    for bad in ([1, 2, 3, 2], [1, 2, 2, 4], [1, 2, 2]):
        with pytest.raises(VerificationError):
            sb.verify_output(inp, np.array(bad, dtype=np.int64))


def test_gen_data_matches_reference(golden):
    for g in golden["gen_data"]:
        assert oracle.fingerprint(sb.gen_data(g["n"], g["seed"])) == int(g["fp"])


def test_gpu_run_benchmark_report_and_trace(tmp_path):
    """bench::run_benchmark's GPU twin: verified report, one compute event per
    rank plus the root merge, exports in the reference's formats."""
    import json

    from paper_1105_6040_b200 import report as R
    rows, reps = R.experiment1(["merge", "quick"], [1 << 16, 5000], [1, 3, 4], [2], seed=3,
                               repetitions=3)
    assert len(rows) == 6
    for row, rep in zip(rows, reps):
        f = row.split(",")
        assert f[0] == rep.config.algorithm and int(f[1]) == rep.config.n
        assert float(f[4]) > 0 and rep.wall_seconds > 0
        kinds = sorted((e.rank, e.kind) for e in rep.world.trace)
        assert kinds.count((0, "gather")) == 1
        assert sum(1 for _, k in kinds if k == "compute") == rep.config.procs
    path = str(tmp_path / "trace.jsonl")
    R.emit_trace(reps[2], path)
    lines = open(path).read().splitlines()
    assert all(json.loads(l)["run_id"] == R.run_id(reps[2].config) for l in lines)
    summ = json.load(open(path + ".summary.json"))
    assert summ["procs"] == 4 and len(summ["ranks"]) == 4


@pytest.mark.parametrize("dt", ["uint32", "uint64", "int32"])
def test_verify_output_device_keys(dt):
    """verify_output on device tensors of every key type: the exact check is
    an independent sort (torch.sort through an order-preserving signed view
    for unsigned keys), so a high-bit key must land last."""
    import torch
    tdt = getattr(torch, dt)
    npdt = np.dtype(dt)
    hi = (1 << (8 * npdt.itemsize - 1)) + 5 if dt.startswith("u") else -7
    host = np.array([3, 1, hi, 2], dtype=npdt)
    signed = np.dtype(f"int{8 * npdt.itemsize}")
    inp = torch.from_numpy(host.view(signed)).cuda().view(tdt)
    good = sb._independent_sort(inp)
    sb.verify_output(inp, good)
    bad = good.flip(0)
    with pytest.raises(sb.VerificationError):
        sb.verify_output(inp, bad)


@pytest.mark.parametrize("p", [16, 32, 64])
def test_exp1_grid_largest_sizes(p):
    """The exp1 grid's largest result-verified runs (P/tests/acceptance.cpp:
    235-261): merge and quick at n = 600,000 with up to 64 processes, each
    checked against the oracle as run_benchmark's verify_output does."""
    data = oracle.gen_data(600_000, 1)
    for algo in (sb.Algorithm.merge, sb.Algorithm.quick):
        out = sb.scatter_merge_sort(algo, data, opts(p)).sorted
        assert np.array_equal(np.asarray(out), oracle.sort(data)), (algo, p)
