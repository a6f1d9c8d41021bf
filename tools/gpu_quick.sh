#!/bin/bash
# Quick GPU iteration: permutation + config parity tests, config-2 bench, launch list.
# usage: bash tools/gpu_quick.sh [pytest -k expr] [tag]
K="${1:-perm or config or golden or rejection}"
TAG="${2:-quick}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_build.py 2 2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/agg_ncu.py gpurun_out/launches_$TAG.csv 2 | head -12
