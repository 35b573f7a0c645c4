#!/bin/bash
# Refresh every committed measurement of the round on one B200 (run from the
# repo root on the GPU box, after `make prof tools` here):  bash tools/round_profile.sh r01
#   bench line (no profiler), ncu launch list of the same command, the
#   per-configuration results, the phase split and the CUB comparison.
p=${1:-r01}
o=gpurun_out
python bench.py --steps 10 --warmup 3 > $o/${p}_bench.log 2>&1; echo bench=$?
python bench.py --steps 2 --warmup 3 --no-cpu > $o/${p}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${p}_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu > $o/${p}_ncu_launch.log 2>&1; echo launches=$?
python tools/config_bench.py > $o/${p}_configs.jsonl 2> $o/${p}_configs.err; echo configs=$?
if [ -f paper_1105_6040_b200/lib/libb200sort_prof.so ]; then
  for k in uni zipf asc; do
    B2S_LIB=paper_1105_6040_b200/lib/libb200sort_prof.so python tools/phase_prof.py 268435456 $k
  done > $o/${p}_phase.txt 2>&1; echo phase=$?
fi
[ -x build/cub_compare ] && build/cub_compare > $o/${p}_cub.jsonl 2>&1; echo cub=$?
