#!/bin/bash
# A/B at 4 ranks: fyb_emitq vs fyb_emit in the epoch-range generate step
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518"
for q in 1 0 1 0; do
  CLAIRPLAN_EMITQ=$q timeout 600 $RUN4 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('emitq=$q', round(d['ms_per_step'],3), d['rank0_phases_ms'])"
done
