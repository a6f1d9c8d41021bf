#!/bin/bash
# ncu --set full of selected kernels of one config-C build (run under gpurun)
# usage: bash tools/gpu_ncu_k.sh TAG "regex" [config] [count]
TAG="$1"; K="$2"; C="${3:-4}"; N="${4:-4}"
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:$K" -c $N -o gpurun_out/ncu_$TAG python tools/prof_build.py $C 1 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$TAG.log
