#!/bin/bash
# 4 ranks: sharded parity with the overlapped merge, then A/B of the overlap
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518"
timeout 900 $RUN4 tools/dist_check.py > gpurun_out/distcheck_mo.log 2>&1; echo "dist_check rc=$?"
grep -E "dist_check|ok=False|Error|error" gpurun_out/distcheck_mo.log | head -10
for v in 1 0 1 0; do
  CLAIRPLAN_MERGE_OVERLAP=$v timeout 600 $RUN4 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('overlap=$v', round(d['ms_per_step'],3), d['rank0_phases_ms'])"
done
