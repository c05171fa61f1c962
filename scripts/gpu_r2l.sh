#!/bin/bash
set -u
TAG=${1:-r2l}
OUT=gpurun_out; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -4 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log; tail -2 $OUT/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-sample-s 10 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
python -c "import json;d=json.load(open('$OUT/bench_$TAG.json'));print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['e2e']['verify_plan_s'], d['e2e']['ms_parts'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > $OUT/bench2_$TAG.json 2> $OUT/bench2_$TAG.err
echo "2-rank shared-GPU functional run rc=$?"; cat $OUT/bench2_$TAG.json | head -c 600; echo; tail -3 $OUT/bench2_$TAG.err
