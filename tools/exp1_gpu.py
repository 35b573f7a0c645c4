"""The reference's experiment 1 (time vs process count, P/src/bench.cpp:224-254)
on the GPU, next to the reference library's own CPU run of the same grid
(oracle/_ref, when built): one CSV in the reference's exp1 format, plus the
GPU traces in its JSONL format.

  python tools/exp1_gpu.py [--n 1048576] [--procs 1,2,4,8] [--cores 4] [--reps 3]
                           [--out profiles/r02_exp1] [--cpu]
                           [--devices 0,1,2,3,4,5,6,7 | --emulate]

Default: m processes = m partitions of the single-GPU partitioned sort. With
--devices (or --emulate: every rank on device 0), m processes = m GPU ranks
of the multi-GPU sample sort behind the C ABI (b2s_sample_sort).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1105_6040_b200 import report as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--procs", default="1,2,4,8")
    ap.add_argument("--cores", default="4")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--algorithms", default="merge,quick")
    ap.add_argument("--out", default=None)
    ap.add_argument("--cpu", action="store_true", help="also run the reference library's grid")
    ap.add_argument("--devices", default=None, help="rank -> GPU list for the multi-GPU grid")
    ap.add_argument("--emulate", action="store_true", help="multi-GPU grid, every rank on GPU 0")
    a = ap.parse_args()
    algos = a.algorithms.split(",")
    procs = [int(x) for x in a.procs.split(",")]
    cores = [int(x) for x in a.cores.split(",")]
    if a.devices or a.emulate:
        devs = [int(x) for x in a.devices.split(",")] if a.devices else [0] * max(procs)
        label = "b200_multi" + ("_emulated" if len(set(devs)) < len(devs) else "")
        rows, reps = [], []
        for algo in algos:
            for m in procs:
                for k in cores:
                    rep = R.run_benchmark_multi(R.RunConfig(algo, a.n, m, k, 1, "wall", a.reps), devs)
                    rows.append(R.exp1_csv_row(rep))
                    reps.append(rep)
    else:
        label = "b200"
        rows, reps = R.experiment1(algos, [a.n] * len(algos), procs, cores, 1, a.reps)
    lines = ["device," + R.EXP1_CSV_HEADER] + [label + "," + r for r in rows]
    if a.cpu:
        import oracle
        for algo in algos:
            for m in procs:
                for k in cores:
                    csv, _, _ = oracle.ref_run_benchmark(algo, a.n, m, k, 1, "wall", a.reps)
                    lines.append("cpu_reference," + csv)
    print("\n".join(lines))
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out + ".csv", "w") as f:
            f.write("\n".join(lines) + "\n")
        for rep in reps:
            R.emit_trace(rep, f"{a.out}_{rep.config.algorithm}_m{rep.config.procs}_k{rep.config.cores}.jsonl")


if __name__ == "__main__":
    main()
