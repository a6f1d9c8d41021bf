#!/bin/bash
bash tools/gpu_sweep_env.sh CLAIRPLAN_FYB_THREADS "128 256 512"
for W in 1 2 3 6; do CLAIRPLAN_CSR_WINDOWS=$W CLAIRPLAN_DENSE=0 timeout 300 python tools/prof_shard_streams.py 2 3 4 2>&1 | tail -1 | sed "s/^/windows=$W /"; done
