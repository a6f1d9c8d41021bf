#!/bin/bash
# Multi-GPU check (run under gpurun --gpus N): parity of the sharded build, then bench lines.
# usage: bash tools/gpu_dist.sh N [tag] [configs]
N="${1:-2}"; TAG="${2:-dist}"; CFGS="${3:-2}"
mkdir -p gpurun_out
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517"
timeout 900 $RUN tools/dist_check.py > gpurun_out/distcheck_$TAG.log 2>&1; echo "dist_check rc=$?"
grep -E "dist_check|ok=False|Error|error" gpurun_out/distcheck_$TAG.log | head -20
for c in $CFGS; do
  timeout 900 $RUN bench.py --gpus $N --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_${TAG}_c$c.log 2>&1; echo "bench c$c rc=$?"
  tail -1 gpurun_out/bench_${TAG}_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['stages_ms'].items()})"
done
