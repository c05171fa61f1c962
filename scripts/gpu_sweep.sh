#!/bin/bash
# GPU tests + default bench + scheduler-knob sweep around the defaults.
# Usage: bash scripts/gpu_sweep.sh TAG ["ENV=.." ...]
set -u
TAG=${1:-sw}; shift || true
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
bash scripts/gpu_ab.sh $TAG "$@"
