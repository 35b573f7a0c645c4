#!/bin/bash
# Refresh every committed measurement of the round on one B200 (run from the
# repo root on the GPU box, after `make all tools` here):  bash tools/round_profile.sh r02
#   bench line (no profiler), ncu launch list of the same command, DRAM bytes
#   of one cfg3 onesweep pass (2^31 int32, 32-bit look-back words), one
#   `ncu --set full` capture of that pass, the per-configuration results and
#   the CUB comparison.
p=${1:-r02}
o=gpurun_out
python bench.py --steps 10 --warmup 3 > $o/${p}_bench.log 2>&1; echo bench=$?
python bench.py --steps 2 --warmup 3 --no-cpu > $o/${p}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${p}_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu > $o/${p}_ncu_launch.log 2>&1; echo launches=$?
K='regex:onesweep_kernel<unsigned int, \(bool\)0, unsigned int, \(int\)512, \(int\)24, \(int\)2, \(int\)2>'
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -s 6 -c 1 \
    -o $o/${p}_onesweep_cfg3 python bench.py --steps 2 --warmup 3 --no-cpu > $o/${p}_ncu_full.log 2>&1; echo full=$?
python tools/config_bench.py > $o/${p}_configs.jsonl 2> $o/${p}_configs.err; echo configs=$?
[ -x build/cub_compare ] && build/cub_compare > $o/${p}_cub.jsonl 2>&1; echo cub=$?
