for c in 0 4 5 6; do echo "cfg $c"; B2S_ONESWEEP_CFG=$c timeout 120 python tools/prof_sort.py --n 268435456 --iters 3 2>&1 | tail -1; done > gpurun_out/run.log 2>&1
B2S_ONESWEEP_CFG=4 timeout 600 python -m pytest tests/test_gpu_sort.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest4=$? >> gpurun_out/run.log; tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/run.log
B2S_ONESWEEP_CFG=4 B2S_LIB=paper_1105_6040_b200/lib/libb200sort_prof.so python tools/phase_prof.py >> gpurun_out/run.log 2>&1
