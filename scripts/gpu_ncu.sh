#!/bin/bash
# One ncu --set full capture of eval_kernel from a short bench run.
# Usage: bash scripts/gpu_ncu.sh TAG [ENV=..]
set -u
TAG=${1:-n}; shift || true
OUT=gpurun_out
mkdir -p $OUT
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 2 -c 1 \
    -o $OUT/eval_$TAG -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full_$TAG.log 2>&1
tail -2 $OUT/ncu_full_$TAG.log
