#!/bin/bash
# Config-2 bench over bucketed-shuffle geometries: "lgTB:lgTS:threads"
DEF="9:14:256 10:13:256 10:14:256 10:13:512 10:14:512 11:13:512 9:14:256"
for c in ${1:-$DEF}; do
  IFS=: read tb ts th <<< "$c"
  CLAIRPLAN_FY_LGTB=$tb CLAIRPLAN_FY_LGTS=$ts CLAIRPLAN_FYB_THREADS=$th timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), round(d['stages_ms']['permutations+streams'],3))"
done
