#!/bin/bash
# ncu --set full captures of the top plan kernels (config 2), one launch each (run under gpurun).
# usage: bash tools/gpu_ncu_full.sh "<kernel regex>" <tag> [config]
set -x
K="${1:-regex:fyb_block|fyb_emit|holder_tile|seg_write_kernel2}"
TAG="${2:-full}"
C="${3:-2}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k "$K" -c 8 \
  -o gpurun_out/ncu_$TAG python tools/prof_build.py $C 1 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
tail -5 gpurun_out/ncu_$TAG.log
