#!/bin/bash
# A/B: grid sizing (CTAs per SM) of sample_tile and seg_allfit
bash tools/gpu_sweep_env.sh CLAIRPLAN_GRID_SAMPLE "8 4 6 12 16 8"
bash tools/gpu_sweep_env.sh CLAIRPLAN_GRID_ALLFIT "8 4 16 32 8"
