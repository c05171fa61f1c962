#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python scripts/per_program_time.py llama3-405b-tp8pp16dp2 > $OUT/perprog_r2k.txt 2>&1; cat $OUT/perprog_r2k.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 3 -c 1 \
    -o $OUT/eval_r2k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full_r2k.log 2>&1
tail -1 $OUT/ncu_full_r2k.log
