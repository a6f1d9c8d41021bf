#!/bin/bash
# Config-2 bench under a sweep of one environment variable: prints ms/step and stage times.
# usage: bash tools/gpu_sweep_env.sh VAR "v1 v2 ..." [config]
VAR="$1"; VALS="$2"; C="${3:-2}"
for v in $VALS; do
  if [ "$v" = "unset" ]; then unset $VAR; else export $VAR="$v"; fi
  timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['stages_ms'].items()})"
done
