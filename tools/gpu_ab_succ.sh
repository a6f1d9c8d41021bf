#!/bin/bash
# A/B: succ preset by memset (default) vs every writer's succ written by fyb_block
bash tools/gpu_sweep_env.sh CLAIRPLAN_SUCC_ALL "0 1 0 1"
CLAIRPLAN_SUCC_ALL=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_succall.csv python tools/prof_build.py 2 2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/agg_ncu.py gpurun_out/launches_succall.csv 2 | head -8
