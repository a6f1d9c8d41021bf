#!/bin/bash
# time + DRAM bytes of one kernel (regex) of a config-C build under several env settings
# usage: bash tools/gpu_ncu_env.sh TAG REGEX C "KV;KV;..."
TAG="$1"; K="$2"; C="$3"; SETS="$4"
mkdir -p gpurun_out
IFS=';' read -ra ARR <<< "$SETS"
i=0
for set in "${ARR[@]}"; do
  ( [ "$set" != "-" ] && for kv in $set; do export "$kv"; done
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k "regex:$K" --csv --log-file gpurun_out/ne_${TAG}_$i.csv python tools/prof_build.py $C 1 > /dev/null 2>&1
    echo "[$set] $(python tools/agg_ncu.py gpurun_out/ne_${TAG}_$i.csv 2>/dev/null | head -3 | tr '\n' ' ')" )
  i=$((i+1))
done
