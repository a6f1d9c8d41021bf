#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "allfit or config or sharded" 2>&1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['stages_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:seg_allfit --csv python tools/prof_build.py 2 1 2>/dev/null | grep seg_allfit | awk -F'","' '{print $(NF-3), $NF}'
