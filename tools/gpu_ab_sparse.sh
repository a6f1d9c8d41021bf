#!/bin/bash
# A/B: sparse_sample grid / occupancy on an emulated 4-way shard (config 2), sparse passes forced
timeout 600 python -m pytest tests -m gpu -x -q -k sharded 2>&1 | tail -1
export CLAIRPLAN_DENSE=0
for c in "8:6" "6:6" "12:6" "5:5" "10:5" "8:6"; do
  IFS=: read g m <<< "$c"
  CLAIRPLAN_GRID_SPARSE=$g CLAIRPLAN_SPARSE_MINB=$m timeout 300 python tools/prof_shard_streams.py 2 5 4 2>&1 | tail -1 | sed "s/^/grid=$g minb=$m /" | cut -c1-140
done
