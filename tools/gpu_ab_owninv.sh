#!/bin/bash
# 2 ranks: sharded parity with the own-epoch inverse rows, then A/B
timeout 600 python -m pytest tests -m gpu -x -q -k sharded 2>&1 | tail -1
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518"
timeout 900 $RUN2 tools/dist_check.py > gpurun_out/distcheck_oi.log 2>&1; echo "dist_check rc=$?"
grep -E "dist_check|ok=False|Error|error" gpurun_out/distcheck_oi.log | head -10
for v in 1 0 1 0; do
  CLAIRPLAN_OWN_INV=$v timeout 600 $RUN2 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('own_inv=$v', round(d['ms_per_step'],3), d['rank0_phases_ms'])"
done
