#!/bin/bash
# A/B variants of the kernel in one box: bench.py (kernel time only) per variant.
# Usage: bash scripts/gpu_ab.sh TAG "ENV=.. ENV=.." ...   (PQW_LIB=variants/x.so selects a build)
set -u
TAG=${1:-ab}; shift || true
OUT=gpurun_out; mkdir -p $OUT
i=0
for v in "$@"; do
  i=$((i+1))
  echo "== variant $i: $v" | tee -a $OUT/ab_$TAG.log
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ab_${TAG}_v$i.json 2> $OUT/ab_${TAG}_v$i.err
  python -c "import json;d=json.load(open('$OUT/ab_${TAG}_v$i.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms'])" 2>&1 | tail -1 | tee -a $OUT/ab_$TAG.log
  grep PQW_PROF $OUT/ab_${TAG}_v$i.err | tail -20 | tee -a $OUT/ab_$TAG.log
done
