#!/bin/bash
# 4-GPU box: sharded parity, N=4 bench lines (config 2 with e2e, config 4), N=2 config 2.
TAG="${1:-d4f}"
mkdir -p gpurun_out
bash tools/gpu_dist.sh 4 $TAG "4"
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518"
timeout 900 $RUN4 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_c2.log 2>&1; echo "bench n4 c2 rc=$?"
tail -1 gpurun_out/bench_${TAG}_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],3), d['e2e'], d['rank0_phases_ms'], d['clocks'])"
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519"
timeout 900 $RUN2 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_n2_c2.log 2>&1; echo "bench n2 c2 rc=$?"
tail -1 gpurun_out/bench_${TAG}_n2_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],3), d['e2e'], d['rank0_phases_ms'])"
