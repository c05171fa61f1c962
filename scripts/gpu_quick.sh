#!/bin/bash
# Quick GPU pass: GPU parity tests, smoke, bench (+ variants given as env strings).
# Usage: bash scripts/gpu_quick.sh TAG ["ENV=.. ENV2=.." ...]
set -u
TAG=${1:-q}; shift || true
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
cat $OUT/smoke_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-sample-s 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
i=0
for v in "$@"; do
  i=$((i+1))
  echo "== variant $v"
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_${TAG}_v$i.json 2> $OUT/bench_${TAG}_v$i.err
  python -c "import json;d=json.load(open('$OUT/bench_${TAG}_v$i.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'])" 2>&1 | tail -1
done
