"""SASS opcode histogram of every kernel in the shipped library
(cuobjdump -sass), so the Blackwell-native instructions each kernel uses are
on record: UBLKCP (cp.async.bulk, TMA bulk copies), SYNCS (mbarrier),
ATOMS (shared atomics), LDGSTS (cp.async), STG.E.EF (streaming stores)...

  python tools/sass_histogram.py [lib.so] > profiles/r02_sass_opcodes.json
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1105_6040_b200", "lib",
                                                         "libb200sort.so")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    kernels = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            kernels[cur][m.group(1)] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True,
                               text=True).stdout.splitlines()
    out = {}
    for (mangled, ops), name in zip(kernels.items(), demangled):
        base = {}
        for op, c in ops.items():
            base[op] = base.get(op, 0) + c
        out[name] = {"instructions": sum(ops.values()),
                     "blackwell": {k: v for k, v in sorted(base.items())
                                   if k.split(".")[0] in ("UBLKCP", "SYNCS", "UTMALDG", "UTMASTG",
                                                          "ATOMS", "LDGSTS", "REDUX", "VOTE",
                                                          "MATCH", "ELECT", "ACQBULK")},
                     "top": dict(ops.most_common(12))}
    json.dump({"library": os.path.relpath(LIB, ROOT), "tool": "cuobjdump -sass (CUDA 12.9)",
               "kernels": out}, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
