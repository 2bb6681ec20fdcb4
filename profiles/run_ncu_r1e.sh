#!/bin/bash
OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:'k_tc_gemm' -s 30 -c 4 \
    -o $OUT/prof_gemm_r1e python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_r1e.log 2>&1
