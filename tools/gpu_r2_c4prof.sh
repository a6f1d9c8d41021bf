#!/bin/bash
# Round-2 baseline: config-4 launch list (time + DRAM bytes) and ncu --set full of the top
# config-4 kernels (run under gpurun).
TAG="${1:-r2base}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt
nproc > gpurun_out/nproc_${TAG}.txt; free -g >> gpurun_out/nproc_${TAG}.txt
timeout 600 python tools/prof_build.py 4 2 > gpurun_out/c4_${TAG}.log 2>&1; echo "c4 build rc=$?"; tail -2 gpurun_out/c4_${TAG}.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv python tools/prof_build.py 4 1 > gpurun_out/ncu_list_${TAG}.log 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:seg_write|holder_tile|fy_link|fy_group|fy_emit|ff_|first_fit|class_write|blk_codes|sample_tile" -c 12 -o gpurun_out/ncu_${TAG}_c4 python tools/prof_build.py 4 1 > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full_${TAG}.log
