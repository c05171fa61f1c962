#!/bin/bash
set -u
TAG=${1:-r2d}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python scripts/pack_bench.py > $OUT/pack_$TAG.log 2>&1; cat $OUT/pack_$TAG.log
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -5 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-sample-s 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
cat $OUT/bench_$TAG.json | python -c "import json,sys;d=json.load(sys.stdin);print(d['value'],d['e2e'])"
bash scripts/gpu_ab.sh $TAG "PQW_LIB=variants/lib_prof.so" "PQW_SLEEP=0" "PQW_SLEEP=100" "PQW_SLEEP=400"
