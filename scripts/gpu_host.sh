#!/bin/bash
# host-path timing (packer / plan create phases) + a default bench line
set -u
TAG=${1:-h}
OUT=gpurun_out; mkdir -p $OUT
PQW_TIMING=1 timeout 900 python scripts/host_timing.py > $OUT/host_timing_$TAG.txt 2>&1
grep -v "PQW_TIMING load" $OUT/host_timing_$TAG.txt | tail -12
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
python -c "import json;d=json.load(open('$OUT/bench_$TAG.json'));e=d['e2e'];print('value',d['value'],'e2e',e['value'],e['verify_plan_s'],e['verify_plan_s_runs'],e['ms_parts'])"
