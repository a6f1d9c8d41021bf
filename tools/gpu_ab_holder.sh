#!/bin/bash
# A/B: holder_tile grid (CTAs per SM) and tile rows in flight
for c in "16:4" "5:4" "10:4" "16:8" "5:8" "16:4"; do
  IFS=: read g t <<< "$c"
  CLAIRPLAN_HOLDER_GRID=$g CLAIRPLAN_HOLDER_TU=$t timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('grid=$g tu=$t', round(d['ms_per_step'],3), round(d['stages_ms']['holder_csr'],3))"
done
