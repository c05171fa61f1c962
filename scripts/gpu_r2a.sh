#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_r2a.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_r2a.log
tail -3 $OUT/pytest_gpu_r2a.log
timeout 600 python bench.py --workload llama3-405b-tp8pp16dp2 --steps 10 --warmup 3 --cpu-sample-s 5 > $OUT/bench_r2a_405b.json 2> $OUT/bench_r2a_405b.err
cat $OUT/bench_r2a_405b.json; tail -3 $OUT/bench_r2a_405b.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 2 -c 1 \
    -o $OUT/eval_r2a_405b -f python bench.py --workload llama3-405b-tp8pp16dp2 --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full_r2a.log 2>&1
tail -2 $OUT/ncu_full_r2a.log
