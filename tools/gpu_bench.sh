#!/bin/bash
# quick bench lines (run under gpurun): usage bash tools/gpu_bench.sh TAG [env assignments...]
TAG="$1"; shift
for kv in "$@"; do export "$kv"; done
mkdir -p gpurun_out
for c in 4 2; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c$c.log 2>&1; echo "bench c$c rc=$?"
tail -1 gpurun_out/bench_${TAG}_c$c.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), d['stages_ms'])" 2>&1 | tail -1
done
