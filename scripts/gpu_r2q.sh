#!/bin/bash
set -u
TAG=${1:-r2q}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python scripts/pack_bench.py > $OUT/pack_$TAG.log 2>&1; cat $OUT/pack_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-sample-s 10 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
python -c "import json;d=json.load(open('$OUT/bench_$TAG.json'));print('405b value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['e2e']['verify_plan_s'], d['e2e']['ms_parts'])"
for w in llama3-8b-tp4pp2dp2-sp deepseek-v3-tp4pp4dp2-ep llama-2l-tp2dp2 "llama3-8b-tp4pp2dp2-sp~wrong_allreduce_scaling"; do
  timeout 900 python bench.py --workload "$w" --steps 10 --warmup 3 --no-cpu-baseline > "$OUT/bench_${TAG}_$w.json" 2> "$OUT/bench_${TAG}_$w.err"
  python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],'value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['e2e']['verify_plan_s'],d['e2e']['verdict'])" "$OUT/bench_${TAG}_$w.json" "$w"
done
