#!/bin/bash
# host-path phase times (PQW_TIMING) on the 405B plan + verify_plan breakdown
set -u
TAG=${1:-h}
OUT=gpurun_out; mkdir -p $OUT
PQW_TIMING=1 timeout 900 python scripts/pack_bench.py > $OUT/pack_bench_$TAG.txt 2>&1
timeout 900 python scripts/e2e_breakdown.py llama3-405b-tp8pp16dp2 > $OUT/e2e_bd_$TAG.txt 2>&1
tail -3 $OUT/e2e_bd_$TAG.txt | cut -c1-300
