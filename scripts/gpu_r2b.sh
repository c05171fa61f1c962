#!/bin/bash
# Round-2 GPU pass: gpu tests, smoke, default bench (405B), reference arm, 8B bench.
set -u
TAG=${1:-r2b}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -5 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
cat $OUT/smoke_$TAG.log | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-sample-s 10 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
cat $OUT/bench_ref_$TAG.json; tail -3 $OUT/bench_ref_$TAG.err
