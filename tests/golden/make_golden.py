"""Writes the golden parity fixtures in tests/golden from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libsortbench_ref.so, which
oracle/build_ref.sh compiles from /root/reference/proj/src):

    python tests/golden/make_golden.py

Every expected output below comes from the unmodified reference library
(parallel::scatter_merge_sort, kernels::*, parallel::merge_split_padded,
bench::gen_data); the case streams replay the reference tests' own seeded
generators through oracle/ref_driver.cpp. Outputs are stored as the
order-sensitive 64-bit fingerprint ``oracle.fingerprint`` (plus full vectors
for the small hand-written KATs), so the fixtures stay small.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ALGO_NAMES = ["bubble", "merge", "quick"]


def _cases(fn, count):
    n = np.zeros(count, dtype=np.uint64)
    p = np.zeros(count, dtype=np.int32)
    a = np.zeros(count, dtype=np.int32)
    s = np.zeros(count, dtype=np.uint64)
    fn(count, n.ctypes.data, p.ctypes.data, a.ctypes.data, s.ctypes.data)
    return n, p, a, s


def scatter_cases(fn, count, cores_of):
    """Case stream -> list of dicts with the reference's output fingerprint."""
    n, p, a, s = _cases(fn, count)
    rows = []
    for i in range(count):
        data = oracle.ref_gen_data(int(n[i]), int(s[i]))
        out, _ = oracle.ref_scatter_merge_sort(data, int(p[i]), ALGO_NAMES[a[i]],
                                               cores=cores_of(i))
        rows.append({"n": int(n[i]), "p": int(p[i]), "algo": ALGO_NAMES[a[i]],
                     "seed": str(int(s[i])), "fp": str(oracle.fingerprint(out))})
    return rows


def main() -> None:
    if not oracle.ref_available():
        oracle.build()
    ref = oracle.ref()

    # acceptance criterion 1 -- P/tests/acceptance.cpp:121-157
    acc = scatter_cases(ref.ref_acceptance1_cases, 1000, lambda i: 1 + (i % 2))
    # random oracle equivalence -- P/tests/test_parallel_sort.cpp:330-343
    rnd = scatter_cases(ref.ref_random_oracle_cases, 60, lambda i: 1)

    # gen_data pins -- P/src/bench.cpp:57-71 (plus P/tests/test_bench.cpp:53-64)
    gen = []
    for n, seed in [(0, 7), (5, 42), (5, 43), (10000, 1), (4096, 2024), (1 << 16, 1)]:
        d = oracle.ref_gen_data(n, seed)
        gen.append({"n": n, "seed": seed, "fp": str(oracle.fingerprint(d)),
                    "head": [str(int(x)) for x in d[:5]]})

    # hand-written KATs from the reference tests, expected values from the reference
    kats = []

    def kat_sort(name, vals, p, algo):
        data = np.array(vals, dtype=np.int64)
        out, _ = oracle.ref_scatter_merge_sort(data, p, algo)
        kats.append({"name": name, "input": vals, "p": p, "algo": algo,
                     "expected": [int(x) for x in out]})

    kat_sort("bubble five (test_sort_core.cpp:69-72)", [5, 1, 4, 2, 8], 1, "bubble")
    kat_sort("descending triple (test_sort_core.cpp:76-79)", [3, 2, 1], 1, "bubble")
    kat_sort("merge reverse (test_sort_core.cpp:131-134)", [4, 3, 2, 1], 1, "merge")
    kat_sort("merge duplicates (test_sort_core.cpp:136-141)", [2, 7, 1, 8, 2, 8], 1, "merge")
    kat_sort("quick [3,1,2] (test_sort_core.cpp:162-169)", [3, 1, 2], 1, "quick")
    kat_sort("all equal (test_sort_core.cpp:171-177)", [5, 5, 5, 5], 1, "quick")
    kat_sort("p=1 degenerate (test_parallel_sort.cpp:271-279)", [3, 1, 2], 1, "merge")
    kat_sort("two-process bubble (test_parallel_sort.cpp:281-285)", [4, 3, 2, 1], 2, "bubble")
    kat_sort("empty p=3 (test_parallel_sort.cpp:301-305)", [], 3, "merge")
    kat_sort("int64 extremes", [2**63 - 1, -2**63, 0, -1, 1, -2**63, 2**63 - 1], 3, "merge")

    # merge_runs KATs (test_sort_core.cpp:96-121), via the reference
    def ref_merge_runs(a, b):
        a = np.array(a, dtype=np.int64)
        b = np.array(b, dtype=np.int64)
        out = np.empty(a.size + b.size, dtype=np.int64)
        ref.ref_merge_runs(a.ctypes.data if a.size else 0, a.size,
                           b.ctypes.data if b.size else 0, b.size,
                           out.ctypes.data if out.size else 0)
        return [int(x) for x in out]

    merges = []
    for a, b in [([], [1, 2, 3]), ([1, 2, 3], []), ([1, 3, 5], [2, 4, 6]), ([1, 1], [1])]:
        merges.append({"a": a, "b": b, "expected": ref_merge_runs(a, b)})

    # merge_split_padded examples (test_parallel_sort.cpp:171-199) + seeded pairs
    def ref_msp(mine, mv, theirs, tv, high):
        mine = np.array(mine, dtype=np.int64)
        theirs = np.array(theirs, dtype=np.int64)
        out = np.empty(max(mine.size + mv, 1), dtype=np.int64)
        import ctypes
        nr, nv = ctypes.c_uint64(), ctypes.c_uint64()
        ref.ref_merge_split_padded(mine.ctypes.data if mine.size else 0, mine.size, mv,
                                   theirs.ctypes.data if theirs.size else 0, theirs.size,
                                   tv, int(high), out.ctypes.data, ctypes.addressof(nr),
                                   ctypes.addressof(nv))
        return [int(x) for x in out[: nr.value]], int(nv.value)

    msp = []
    fixed = [([1, 3, 5], 0, [2, 4, 6], 0), ([7], 1, [0, 0], 0), ([0, 0], 0, [7], 1),
             ([5], 2, [], 3), ([], 3, [5], 2), ([1, 2], 0, [0, 0], 1)]
    rng = np.random.default_rng(23)
    for _ in range(200):
        width = int(rng.integers(1, 9))
        av, bv = int(rng.integers(0, width + 1)), int(rng.integers(0, width + 1))
        a = sorted(int(x) for x in rng.integers(0, 6, width - av))
        b = sorted(int(x) for x in rng.integers(0, 6, width - bv))
        fixed.append((a, av, b, bv))
    for a, av, b, bv in fixed:
        for high in (False, True):
            reals, virt = ref_msp(a, av, b, bv, high)
            msp.append({"mine": a, "mine_virt": av, "theirs": b, "theirs_virt": bv,
                        "keep": "high" if high else "low", "reals": reals, "virtuals": virt})

    # the local-kernel oracle stream (test_sort_core.cpp:191-216): inputs + ref outputs
    sizes = np.zeros(250, dtype=np.uint64)
    values = np.zeros(250 * 512, dtype=np.int64)
    ref.ref_kernel_oracle_cases(250, sizes.ctypes.data, values.ctypes.data)
    total = int(sizes.sum())
    values = values[:total]
    expected = []
    off = 0
    for s in sizes:
        s = int(s)
        blk = values[off: off + s].copy()
        for algo in (0, 1, 2):
            b2 = blk.copy()
            if s:
                ref.ref_kernel_sort(algo, b2.ctypes.data, s)
            if algo == 1:
                expected.append(str(oracle.fingerprint(b2)))
            else:
                assert np.array_equal(b2, np.sort(blk))
        off += s
    np.savez_compressed(os.path.join(OUT, "kernel_oracle.npz"), sizes=sizes,
                        values=values.astype(np.int8))

    # config-scale pins: cfg1 (N=2^20 int32 = z>>33, p=4) through the reference
    cfg = []
    for n, p, shift in [(1 << 20, 4, 33), (1 << 18, 8, 33), (1 << 20, 4, 0)]:
        z = oracle.ref_gen_data(n, 1).view(np.uint64)
        keys = (z >> np.uint64(shift)).astype(np.int64) if shift else z.view(np.int64)
        out, _ = oracle.ref_scatter_merge_sort(keys, p, "merge", cores=p)
        cfg.append({"n": n, "p": p, "seed": 1, "shift": shift,
                    "fp": str(oracle.fingerprint(out))})

    golden = {
        "generator": "tests/golden/make_golden.py (reference library: oracle/_ref)",
        "acceptance1": acc,
        "random_oracle": rnd,
        "gen_data": gen,
        "kats": kats,
        "merge_runs": merges,
        "merge_split_padded": msp,
        "kernel_oracle_merge_fp": expected,
        "config_pins": cfg,
    }
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(golden, f, indent=0)
    print("wrote", os.path.join(OUT, "golden.json"))

    # report / trace export pins (bench.cpp's run_id, format_double, exp1 row,
    # trace JSONL and summary): counted mode is bit-deterministic
    rng = np.random.default_rng(77)
    ids = []
    for algo in ("bubble", "merge", "quick"):
        for n, p, k, seed, mode, reps in [(1 << 20, 4, 4, 1, "wall", 3), (1000, 1, 1, 7, "counted", 1),
                                          (0, 8, 2, 123, "wall", 1), (1 << 31, 8, 8, 1, "counted", 5)]:
            ids.append({"algorithm": algo, "n": n, "procs": p, "cores": k, "seed": seed,
                        "mode": mode, "repetitions": reps,
                        "run_id": oracle.ref_run_id(algo, n, p, k, seed, mode, reps)})
    vals = [0.0, -0.0, 1.0, 0.5, 100.0, 1e5, 1e6, 123456.7, 999999.5, 1234567.0, 1e-4, 1e-5,
            1.25e-5, 3062828.0, 0.213485530554838, 1.0 / 3.0, 2.0e7 / 3.0, 1e21, 5e-324,
            1.7976931348623157e308, -2.5, -1234567.0]
    vals += [float(x) for x in rng.uniform(-1e3, 1e3, 40)]
    vals += [float(10.0 ** e) * float(m) for e, m in zip(rng.integers(-12, 14, 80), rng.uniform(1, 10, 80))]
    vals += [float(x) for x in rng.integers(0, 1 << 40, 20)]
    chars = [{"v": repr(v), "s": oracle.ref_to_chars_general(v)} for v in vals]
    exports = []
    for algo, n, p, k in [("merge", 4096, 4, 2), ("quick", 3000, 3, 3), ("bubble", 500, 2, 1)]:
        csv, trace, summary = oracle.ref_run_benchmark(algo, n, p, k, 1, "counted", 1)
        exports.append({"algorithm": algo, "n": n, "procs": p, "cores": k, "seed": 1,
                        "mode": "counted", "repetitions": 1, "csv": csv, "trace": trace,
                        "summary": summary})
    with open(os.path.join(OUT, "report_golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference library: oracle/_ref)",
                   "run_ids": ids, "to_chars": chars, "exports": exports}, f, indent=0)
    print("wrote", os.path.join(OUT, "report_golden.json"))


if __name__ == "__main__":
    main()
