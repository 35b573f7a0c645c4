"""The reference's CPU timings for every BASELINE configuration, as SURVEY.md
section 8(d) specifies them (run on the GPU box's host, beside the GPU runs):
parallel::scatter_merge_sort of the reference library (oracle/_ref), wall
mode, median of 3 reps of the world's wall seconds (run_benchmark's
semantics, P/src/bench.cpp:106-169), on bounded samples of each workload
widened to int64 (the reference's only key type):

  cfg1  2^20 int32 keys, p = k = 4, merge and quick (bubble: ~3.4e10
        comparisons per rank, excluded)
  cfg2  2^24-key sample of full-range uint32, merge, p = 1 and p = k = nproc
  cfg3  2^24-key sample of int32 in [0, 2^31), merge, p in {1,2,4,8} and nproc
  cfg4  2^24-key samples of (a) Zipf(1.2) (b) ascending (c) descending
        (d) all-equal, merge only (quick is quadratic on (a) and (d)),
        p = k = nproc
  cfg5  no reference key/value path: a single-threaded stable sort of
        2^22 (uint64 key, uint32 index) pairs, the C restatement (labelled)

  python tools/cpu_baselines.py [--out profiles/r01_cpu_baselines.jsonl]
"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def timed_ref(data, p, k, algo, reps=3):
    times = []
    out = None
    for _ in range(reps):
        out, secs = oracle.ref_scatter_merge_sort(data, p, algo, cores=k, wall=True)
        times.append(secs)
    if not (out[1:] >= out[:-1]).all():
        raise RuntimeError("reference output unsorted")
    return sorted(times)[(len(times) - 1) // 2]


def zipf(z, s=1.2, values=1 << 20):
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    w = np.arange(1, values + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return np.minimum(np.searchsorted(cdf, u), values - 1).astype(np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--sample", type=int, default=1 << 24)
    a = ap.parse_args()
    if not oracle.ref_available():
        sys.exit("oracle/_ref is not built (bash oracle/build_ref.sh)")
    nproc = os.cpu_count() or 1
    host = {"nproc": nproc, "cpu": cpu_model()}
    rows = []

    def rec(cfg, case, n, p, k, algo, secs, kind="reference"):
        row = {"config": cfg, "case": case, "n": n, "p": p, "k": k, "algorithm": algo,
               "seconds": secs, "keys_per_s": n / secs, "kind": kind, **host}
        rows.append(row)
        print(json.dumps(row), flush=True)

    z20 = oracle.gen_data_np(1 << 20, 1)
    d1 = (z20 >> np.uint64(33)).astype(np.int64)
    for algo in ("merge", "quick"):
        rec("cfg1", "2^20 int32 (z >> 33)", d1.size, 4, 4, algo, timed_ref(d1, 4, 4, algo))

    ns = a.sample
    z = oracle.gen_data_np(ns, 1)
    d2 = (z >> np.uint64(32)).astype(np.int64)
    for p in (1, nproc):
        rec("cfg2", f"sample of 2^28: {ns} uint32 (z >> 32)", ns, p, p, "merge", timed_ref(d2, p, p, "merge"))
    d3 = (z >> np.uint64(33)).astype(np.int64)
    for p in sorted({1, 2, 4, 8, nproc}):
        rec("cfg3", f"sample of 2^31: {ns} int32 (z >> 33)", ns, p, min(p, nproc), "merge",
            timed_ref(d3, p, min(p, nproc), "merge"))
    cases = {"(a) Zipf s=1.2 over 2^20 values": zipf(z), "(b) ascending": np.arange(ns, dtype=np.int64),
             "(c) descending": np.arange(ns - 1, -1, -1, dtype=np.int64),
             "(d) all equal": np.full(ns, 7, dtype=np.int64)}
    for name, d in cases.items():
        rec("cfg4", f"sample of 2^27: {ns} keys {name}", ns, nproc, nproc, "merge",
            timed_ref(d, nproc, nproc, "merge"))
    n5 = 1 << 22
    k5 = oracle.gen_data_np(n5, 1)
    v5 = np.arange(n5, dtype=np.uint32)
    t0 = time.perf_counter()
    oracle.stable_sort_kv(k5, v5)
    rec("cfg5", f"sample of 2^28: {n5} (uint64 key, uint32 index) pairs", n5, 1, 1,
        "stable merge sort (C restatement; the reference has no key/value path)",
        time.perf_counter() - t0, kind="port")
    if a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
