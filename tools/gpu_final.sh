#!/bin/bash
# Measurement pass (run under gpurun): bench lines (config 2 full, config 4), launch list and
# ncu --set full captures of the top kernels of config 2; summaries into gpurun_out/.
TAG="${1:-final}"
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_c2.log 2>&1; echo "bench c2 rc=$?"
tail -1 gpurun_out/bench_${TAG}_c2.log | cut -c1-400
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c4.log 2>&1; echo "bench c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_${TAG}_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/bench_${TAG}_ref.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c2.csv python tools/prof_build.py 2 2 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:fyb_block|fyb_emit|holder_tile|sample_tile|seg_allfit|fyb_tile" -c 6 -o gpurun_out/ncu_${TAG} python tools/prof_build.py 2 1 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu full rc=$?"
