"""CPU: pins the C restatement (oracle/oracle.c) against the reference's own
outputs (tests/golden, generated from oracle/_ref) and, where the compiled
reference is present, against the reference library directly."""
import numpy as np
import pytest

import oracle


def test_gen_data_matches_reference_pins(golden):
    for g in golden["gen_data"]:
        d = oracle.gen_data(g["n"], g["seed"])
        assert oracle.fingerprint(d) == int(g["fp"])
        assert [str(int(x)) for x in d[:5]] == g["head"]
        # vectorised numpy form of the same stream
        assert np.array_equal(oracle.gen_data_np(g["n"], g["seed"]).view(np.int64), d)


def test_gen_data_window_is_a_slice():
    full = oracle.gen_data(1000, 9)
    assert np.array_equal(oracle.gen_data(300, 9, first=200), full[200:500])


def test_plan_partition_reference_cases():
    # P/tests/test_parallel_sort.cpp:45-58
    assert oracle.plan_partition(200000, 8) == [25000] * 8
    assert oracle.plan_partition(5, 1) == [5]
    assert oracle.plan_partition(8, 3) == [3, 3, 2]
    with pytest.raises(ValueError):
        oracle.plan_partition(4, 0)


def test_acceptance1_port_matches_reference(golden):
    """Criterion 1 (P/tests/acceptance.cpp:121-157): the port's
    scatter_merge_sort reproduces the reference output on all 1000 cases."""
    for c in golden["acceptance1"]:
        data = oracle.gen_data(c["n"], int(c["seed"]))
        out = oracle.scatter_merge_sort(data, c["p"])
        assert oracle.fingerprint(out) == int(c["fp"]), c
        assert oracle.fingerprint(oracle.sort(data)) == int(c["fp"])


def test_random_oracle_port_matches_reference(golden):
    for c in golden["random_oracle"]:
        data = oracle.gen_data(c["n"], int(c["seed"]))
        assert oracle.fingerprint(oracle.scatter_merge_sort(data, c["p"])) == int(c["fp"])


def test_kats(golden):
    for k in golden["kats"]:
        data = np.array(k["input"], dtype=np.int64)
        assert oracle.scatter_merge_sort(data, k["p"]).tolist() == k["expected"], k["name"]


def test_merge_runs_tie_rule(golden):
    for m in golden["merge_runs"]:
        out = oracle.merge_runs(np.array(m["a"], dtype=np.int64), np.array(m["b"], dtype=np.int64))
        assert out.tolist() == m["expected"]


def test_merge_split_padded(golden):
    for c in golden["merge_split_padded"]:
        reals, virt = oracle.merge_split_padded(c["mine"], c["mine_virt"], c["theirs"],
                                                c["theirs_virt"], c["keep"] == "high")
        assert reals.tolist() == c["reals"] and virt == c["virtuals"], c


def test_kernel_oracle_stream(golden):
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "kernel_oracle.npz"))
    sizes, values = z["sizes"], z["values"].astype(np.int64)
    off = 0
    for s, fp in zip(sizes, golden["kernel_oracle_merge_fp"]):
        s = int(s)
        assert oracle.fingerprint(oracle.sort(values[off: off + s])) == int(fp)
        off += s


def test_config_pins_port(golden):
    for c in golden["config_pins"]:
        z = oracle.gen_data(c["n"], c["seed"]).view(np.uint64)
        keys = (z >> np.uint64(c["shift"])).astype(np.int64) if c["shift"] else z.view(np.int64)
        assert oracle.fingerprint(oracle.scatter_merge_sort(keys, c["p"])) == int(c["fp"])


def test_exhaustive_01_small():
    """P/tests/test_parallel_sort.cpp:314-328 (n <= 8, p in {2,3,4})."""
    for p in (2, 3, 4):
        for n in range(9):
            for mask in range(1 << n):
                data = np.array([(mask >> i) & 1 for i in range(n)], dtype=np.int64)
                assert oracle.scatter_merge_sort(data, p).tolist() == sorted(data.tolist())


def test_stable_kv_restatement():
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 50, 5000).astype(np.uint64)
    vals = np.arange(5000, dtype=np.uint32)
    k, v = oracle.stable_sort_kv(keys, vals)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(k, keys[order]) and np.array_equal(v, vals[order])


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_port_vs_reference_library_direct():
    rng = np.random.default_rng(11)
    for _ in range(50):
        n = int(rng.integers(0, 3000))
        p = int(rng.choice([1, 2, 3, 4, 5, 8]))
        data = oracle.gen_data(n, int(rng.integers(0, 2**63)))
        ref_out, _ = oracle.ref_scatter_merge_sort(data, p, "merge")
        assert np.array_equal(oracle.scatter_merge_sort(data, p), ref_out)
