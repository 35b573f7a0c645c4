#!/bin/bash
# One `ncu --set full` capture of the headline onesweep pass (regular kernel,
# RANK 2, u32 512x24 tiles) on the bench workload.  Usage (on the GPU box):
#   bash tools/ncu_capture.sh gpurun_out/r01_onesweep
out=${1:-gpurun_out/onesweep}
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:onesweep_kernel<unsigned int, \(bool\)0, unsigned int, \(int\)512, \(int\)24, \(int\)2, \(int\)2>' \
    -s 8 -c 1 -o "$out" python bench.py --steps 2 --warmup 3 --no-cpu
