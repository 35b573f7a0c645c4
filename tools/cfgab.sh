#!/bin/bash
# A/B of the onesweep tile configurations (B2S_ONESWEEP_CFG) per key type on
# 2^28 keys: two 512-thread CTAs per SM vs one 1024-thread CTA (the default
# for 8-byte keys + payload only).
# Run on the GPU box from the repo root; results in gpurun_out/cfgab.log.
o=gpurun_out/cfgab.log; : > $o
for dt in u32 u64; do for v in "" "--vals"; do for c in 0 1024; do
  cfg=0; if [ $c = 1024 ]; then if [ $dt = u32 ] && [ -z "$v" ]; then cfg=11; elif [ $dt = u64 ] && [ -n "$v" ]; then cfg=0; else cfg=2; fi; else if [ $dt = u64 ] && [ -n "$v" ]; then cfg=3; fi; fi
  echo "== $dt $v cfg=$cfg" >> $o
  B2S_ONESWEEP_CFG=$cfg python tools/prof_sort.py --n 268435456 --dtype $dt $v --iters 4 2>&1 | tail -n 1 >> $o
done; done; done
