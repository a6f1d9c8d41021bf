#!/bin/bash
# One GPU round: gpu tests, config-2 and config-4 bench lines, config-2 ncu launch list (run under gpurun).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_c2.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench4 rc=$?"
tail -1 gpurun_out/bench_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_build.py 2 2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
