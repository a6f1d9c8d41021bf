#!/bin/bash
# Iteration pass (run under gpurun): GPU parity suite, config-4/2 bench lines (no CPU leg),
# config-4 ncu launch list with DRAM bytes.  usage: bash tools/gpu_iter.sh TAG [pytest-args]
TAG="${1:-it}"; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${@} > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
for c in 4 2; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c$c.log 2>&1; echo "bench c$c rc=$?"
tail -1 gpurun_out/bench_${TAG}_c$c.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), d['stages_ms'])" 2>&1 | tail -1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv python tools/prof_build.py 4 1 > gpurun_out/ncu_list_${TAG}.log 2>&1; echo "ncu list rc=$?"
python tools/agg_ncu.py gpurun_out/launches_${TAG}_c4.csv | head -25
