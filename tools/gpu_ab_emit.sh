#!/bin/bash
# A/B: fyb_emitq (work-list chase) at 4/5 CTAs per SM vs fyb_emit; permutation parity first
timeout 900 python -m pytest tests -m gpu -x -q -k "perm or golden or rejection or config" 2>&1 | tail -2
for c in "1:5" "1:4" "0:5" "1:5" "0:5"; do
  IFS=: read q m <<< "$c"
  CLAIRPLAN_EMITQ=$q CLAIRPLAN_EMITQ_MINB=$m timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('emitq=$q minb=$m', round(d['ms_per_step'],3), round(d['stages_ms']['permutations+streams'],3))"
done
for c in "1:5" "1:4"; do
  IFS=: read q m <<< "$c"
  CLAIRPLAN_EMITQ=$q CLAIRPLAN_EMITQ_MINB=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:emit --csv python tools/prof_build.py 2 1 2>/dev/null | grep -E "gpu__time" | tail -1
done
