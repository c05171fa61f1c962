#!/bin/bash
# Final round pass: gpu tests, smoke, default bench + reference arm, all BASELINE
# configs, 2-rank functional run, kernel capture.
set -u
TAG=${1:-final}
OUT=gpurun_out; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log; tail -2 $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
python -c "import json;d=json.load(open('$OUT/bench_$TAG.json'));print('405b value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['e2e']['verify_plan_s'],d['e2e']['verify_plan_s_runs'])"
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
python -c "import json;d=json.load(open('$OUT/bench_ref_$TAG.json'));print('ref value',d['value'],'e2e',d['e2e']['value'],d['e2e']['verify_plan_s'])"
for w in llama-2l-tp2dp2 llama3-8b-tp4pp2dp2-sp "llama3-8b-tp4pp2dp2-sp~misordered_concat" deepseek-v3-tp4pp4dp2-ep; do
  timeout 900 python bench.py --workload "$w" --steps 10 --warmup 3 --no-cpu-baseline > "$OUT/bench_${TAG}_$w.json" 2> "$OUT/bench_${TAG}_$w.err"
  python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],'value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['e2e']['verify_plan_s'],d['e2e']['verdict'])" "$OUT/bench_${TAG}_$w.json" "$w"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > $OUT/bench2_$TAG.json 2> $OUT/bench2_$TAG.err
echo "2-rank rc=$?"; python -c "import json;d=json.load(open('$OUT/bench2_$TAG.json'));print('2rank value',d['value'],'e2e',d['e2e']['value'],d['e2e']['verify_plan_s'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:eval_kernel -c 30 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 3 -c 1 \
    -o $OUT/eval_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full_$TAG.log 2>&1
tail -1 $OUT/ncu_full_$TAG.log
