#!/bin/bash
# Emulated per-rank sharded builds (sparse and dense sample-major passes) + launch lists.
for G in ${1:-"4 8"}; do
  for D in 0 1; do
    export CLAIRPLAN_DENSE=$D  # 0: sparse passes forced, 1: dense passes forced
    timeout 300 python tools/prof_shard_streams.py 2 3 $G 2>&1 | tail -1 | sed "s/^/dense=$D /"
  done
  export CLAIRPLAN_DENSE=0
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_ss$G.csv python tools/prof_shard_streams.py 2 2 $G > /dev/null 2>&1
  python tools/agg_ncu.py gpurun_out/launches_ss$G.csv 2 2>/dev/null | grep -v "fyb_" | head -14
done
