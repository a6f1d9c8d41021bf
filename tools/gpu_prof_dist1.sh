#!/bin/bash
# Single-GPU run of the sharded (streams) build: stage timing + ncu launch list.
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29519"
timeout 600 $RUN tools/prof_dist.py 2 4 2>&1 | grep "build ms"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_dist1.csv $RUN tools/prof_dist.py 2 2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/agg_ncu.py gpurun_out/launches_dist1.csv 2 2>/dev/null | head -16
