#!/bin/bash
# Full GPU suite, then the measurement pass (tools/gpu_final.sh TAG)
TAG="${1:-final}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_${TAG}.log
bash tools/gpu_final.sh "$TAG"
