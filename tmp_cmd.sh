timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/run.log
tail -15 gpurun_out/pytest_gpu.log >> gpurun_out/run.log
for c in 0 1 2 3; do echo "cfg $c"; B2S_ONESWEEP_CFG=$c timeout 120 python tools/prof_sort.py --n 268435456 --iters 3 2>&1 | tail -1; done >> gpurun_out/run.log 2>&1
for c in 0 1; do echo "cfg $c u64"; B2S_ONESWEEP_CFG=$c timeout 120 python tools/prof_sort.py --n 134217728 --dtype u64 --iters 2 2>&1 | tail -1; echo "cfg $c u64 kv"; B2S_ONESWEEP_CFG=$c timeout 120 python tools/prof_sort.py --n 134217728 --dtype u64 --vals --iters 2 2>&1 | tail -1; echo "cfg $c u32 kv"; B2S_ONESWEEP_CFG=$c timeout 120 python tools/prof_sort.py --n 268435456 --dtype u32 --vals --iters 2 2>&1 | tail -1; done >> gpurun_out/run.log 2>&1
