#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
PQW_LIB=variants/chunk16.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_workload_parity.py -m gpu -x -q -k "bit_exact or matches_oracle or edge" > $OUT/pytest_c16.log 2>&1; echo "rc=$?" >> $OUT/pytest_c16.log; tail -2 $OUT/pytest_c16.log
bash scripts/gpu_ab.sh r2v "PQW_LIB=variants/chunk32.so" "PQW_LIB=variants/chunk16.so" "PQW_LIB=variants/chunk16.so PQW_FAST_SLOTS=1620" "PQW_LIB=variants/chunk32.so"
