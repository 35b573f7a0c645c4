for c in 0 1 3; do echo "cfg $c"; B2S_ONESWEEP_CFG=$c timeout 120 python tools/prof_sort.py --n 268435456 --iters 3 2>&1 | tail -1; done > gpurun_out/run.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sort.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/run.log
