#!/bin/bash
# N ranks: sharded parity incl. the fused peer-memory exchange, then A/B streams vs p2p
N="${1:-2}"
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518"
timeout 900 $RUN tools/dist_check.py > gpurun_out/distcheck_p2p$N.log 2>&1; echo "dist_check rc=$?"
grep -E "dist_check|ok=False|Error|error|not taken" gpurun_out/distcheck_p2p$N.log | head -10
for m in p2p streams p2p streams; do
  CLAIRPLAN_DIST_MODE=$m timeout 600 $RUN bench.py --gpus $N --steps 10 --warmup 3 --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode=$m', round(d['ms_per_step'],3), d['rank0_phases_ms'])"
done
