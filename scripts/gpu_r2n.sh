#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
PQW_LIB=variants/mirror_u2.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_workload_parity.py -m gpu -x -q -k "bit_exact or matches_oracle or edge" > $OUT/pytest_u2.log 2>&1; echo "rc=$?" >> $OUT/pytest_u2.log; tail -3 $OUT/pytest_u2.log
bash scripts/gpu_ab.sh r2n "PQW_LIB=variants/mirror.so" "PQW_LIB=variants/mirror_u2.so" "PQW_LIB=variants/mirror.so" "PQW_LIB=variants/mirror_u2.so"
