#!/bin/bash
# tests + bench + optional A/B variants
set -u
TAG=${1:-q}; shift || true
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -4 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
python -c "import json;d=json.load(open('$OUT/bench_$TAG.json'));print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['e2e']['verify_plan_s'])"
tail -2 $OUT/bench_$TAG.err
if [ $# -gt 0 ]; then bash scripts/gpu_ab.sh $TAG "$@"; fi
