"""The reference's experiment 1 (time vs process count, P/src/bench.cpp:224-254)
with the GPU partitioned sort, next to the reference library's own CPU run of
the same grid (oracle/_ref, when built): one CSV in the reference's exp1
format, plus the GPU traces in its JSONL format.

  python tools/exp1_gpu.py [--n 1048576] [--procs 1,2,4,8] [--cores 4] [--reps 3]
                           [--out profiles/r01_exp1] [--cpu]
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
    a = ap.parse_args()
    algos = a.algorithms.split(",")
    procs = [int(x) for x in a.procs.split(",")]
    cores = [int(x) for x in a.cores.split(",")]
    rows, reps = R.experiment1(algos, [a.n] * len(algos), procs, cores, 1, a.reps)
    lines = ["device," + R.EXP1_CSV_HEADER] + ["b200," + r for r in rows]
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
