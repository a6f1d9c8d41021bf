#!/bin/bash
# Measurement pass (run under gpurun): default bench line (config 4, CPU baseline, e2e), the
# reference arm, config-2 line, ncu launch lists (config 4 and 2) and ncu --set full of the
# top config-4 kernels.  usage: bash tools/gpu_measure.sh TAG
TAG="${1:-meas}"
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_${TAG}_c4.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_${TAG}_c4.log | cut -c1-300
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_c2.log 2>&1; echo "bench c2 rc=$?"
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_${TAG}_ref.log | cut -c1-300
for c in 4 2; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c$c.csv python tools/prof_build.py $c 1 > /dev/null 2>&1; echo "ncu list c$c rc=$?"
done
timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:fyc_|holder_tile|ff_stats|seg_write3|sample_tile" -c 8 -o gpurun_out/ncu_${TAG}_c4 python tools/prof_build.py 4 1 > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "ncu full rc=$?"
