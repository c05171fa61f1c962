#!/bin/bash
# GPU pass: gpu tests, smoke, default bench (405B), host pack timing, ncu capture of eval_kernel.
set -u
TAG=${1:-r2c}
OUT=gpurun_out; mkdir -p $OUT
nproc > $OUT/host_$TAG.txt; lscpu | grep "Model name" >> $OUT/host_$TAG.txt
timeout 600 python scripts/pack_bench.py > $OUT/pack_$TAG.log 2>&1
cat $OUT/pack_$TAG.log
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -5 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
tail -2 $OUT/smoke_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-sample-s 10 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 3 -c 1 \
    -o $OUT/eval_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full_$TAG.log 2>&1
tail -2 $OUT/ncu_full_$TAG.log
