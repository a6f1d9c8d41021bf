#!/bin/bash
# config-4 shuffle-stage sweep over epoch-batch budgets and shuffle modes (run under gpurun)
mkdir -p gpurun_out
for mode in lists bucket12; do
 for b in 100 200 400 1000 4096; do
  if [ $mode = lists ]; then export CLAIRPLAN_FY=lists; unset CLAIRPLAN_FY_MAXLGTB; else export CLAIRPLAN_FY=bucket; export CLAIRPLAN_FY_MAXLGTB=12; fi
  export CLAIRPLAN_PERM_BUDGET_MB=$b
  timeout 300 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ps_${mode}_$b.log 2>&1
  echo "$mode $b rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/ps_${mode}_$b.log').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), d['stages_ms']['permutations+streams'])" 2>&1)"
 done
done
