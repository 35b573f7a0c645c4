python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:onesweep -s 8 -c 1 -o gpurun_out/bench_onesweep_r01b python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
B2S_LIB=paper_1105_6040_b200/lib/libb200sort_prof.so python tools/phase_prof.py > gpurun_out/phase.log 2>&1
