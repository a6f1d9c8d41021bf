#!/bin/bash
# e2e at N ranks: p2p vs streams exchange
N="${1:-4}"
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518"
for m in p2p streams p2p streams; do
  CLAIRPLAN_DIST_MODE=$m timeout 600 $RUN bench.py --gpus $N --steps 10 --warmup 3 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode=$m', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],2), d['rank0_phases_ms'])"
done
