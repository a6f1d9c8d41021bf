#!/bin/bash
# Config-2 bench over combinations "VAR1=a,VAR2=b ..." (space-separated combos).
# usage: bash tools/gpu_sweep2.sh "A=1,B=2 A=3,B=4" [config]
C="${2:-2}"
for combo in $1; do
  ( IFS=','; for kv in $combo; do export "$kv"; done
    timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$combo', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['stages_ms'].items() if x > 0.01})" )
done
