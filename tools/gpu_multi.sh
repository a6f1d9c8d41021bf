#!/bin/bash
# multi-GPU pass (run under gpurun --gpus G): dist_check (parity) + bench lines at N=G
G="${1:-2}"; TAG="${2:-m}"
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py > gpurun_out/distcheck_${TAG}_g$G.log 2>&1; echo "dist_check rc=$?"; grep -E "dist_check|checksums|ok=False" gpurun_out/distcheck_${TAG}_g$G.log | head -20
for c in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $G --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_g${G}_c$c.log 2>&1; echo "bench c$c rc=$?"
tail -1 gpurun_out/bench_${TAG}_g${G}_c$c.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), d['rank0_phases_ms'], 'e2e', round(d['e2e']['ms_per_step'],1))" 2>&1 | tail -1
done
