#!/bin/bash
# ncu launch lists (time + DRAM bytes) of one build per config (run under gpurun)
# usage: bash tools/gpu_list.sh TAG "configs" [env assignments...]
TAG="$1"; CFGS="${2:-4 2}"; shift 2
for kv in "$@"; do export "$kv"; done
mkdir -p gpurun_out
for c in $CFGS; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c$c.csv python tools/prof_build.py $c 1 > gpurun_out/ncu_list_${TAG}_c$c.log 2>&1; echo "ncu list c$c rc=$?"
python tools/agg_ncu.py gpurun_out/launches_${TAG}_c$c.csv 2>/dev/null | head -14
done
