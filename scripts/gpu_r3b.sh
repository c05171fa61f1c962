#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
PQW_LIB=variants/bens.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_workload_parity.py -m gpu -x -q -k "bit_exact or matches_oracle or edge" > $OUT/pytest_bens.log 2>&1; echo "rc=$?" >> $OUT/pytest_bens.log; tail -2 $OUT/pytest_bens.log
bash scripts/gpu_ab.sh r3b "PQW_LIB=variants/base.so" "PQW_LIB=variants/bens.so" "PQW_LIB=variants/base.so" "PQW_LIB=variants/bens.so"
