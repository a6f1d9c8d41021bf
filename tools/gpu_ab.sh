#!/bin/bash
# A/B sweep of CLAIRPLAN_* knobs on one config (run under gpurun; library built with AB_KNOBS=1)
# usage: bash tools/gpu_ab.sh TAG CONFIG "KV1 KV2;KV3;..."   (";"-separated settings, each a
# space-separated list of assignments; "-" = defaults)
TAG="$1"; C="$2"; SETS="$3"
mkdir -p gpurun_out
IFS=';' read -ra ARR <<< "$SETS"
for set in "${ARR[@]}"; do
  ( [ "$set" != "-" ] && for kv in $set; do export "$kv"; done
    timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.log 2>&1
    echo "[$set] rc=$? $(tail -1 gpurun_out/ab_${TAG}.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), {k: round(v,2) for k,v in d['stages_ms'].items()})" 2>&1 | tail -1)" )
done
