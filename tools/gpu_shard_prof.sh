#!/bin/bash
# Per-rank compute profile of a G-way worker-sharded build emulated on one GPU (handle planning
# 1/G of the workers): ncu launch list per G.
for G in ${1:-8}; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_shard$G.csv python tools/prof_build.py 2 2 $G > gpurun_out/shard$G.log 2>&1; echo "G=$G ncu rc=$?"; tail -1 gpurun_out/shard$G.log
  python tools/agg_ncu.py gpurun_out/launches_shard$G.csv 2 2>/dev/null | head -10
done
