#!/bin/bash
# Config-4 bench: linked-list shuffle (default above F = 2^23) vs bucketed geometries "maxlgTB:lgTB:lgTS"
run() { timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3), {k: round(x,2) for k,x in d['stages_ms'].items()})"; }
run default
for c in ${1:-12:12:14 12:11:14 12:11:15}; do
  IFS=: read mx tb ts <<< "$c"
  CLAIRPLAN_FY_MAXLGTB=$mx CLAIRPLAN_FY_LGTB=$tb CLAIRPLAN_FY_LGTS=$ts run "$c"
done
