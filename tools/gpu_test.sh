#!/bin/bash
# GPU parity tests (run under gpurun): bash tools/gpu_test.sh TAG [quick]
TAG="$1"; MODE="${2:-full}"
mkdir -p gpurun_out
if [ "$MODE" = quick ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "not full_plan and not config5" > gpurun_out/pytest_${TAG}.log 2>&1
else
  timeout 2000 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_${TAG}.log 2>&1
fi
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_${TAG}.log
