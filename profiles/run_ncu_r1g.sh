#!/bin/bash
# r1g: --set full on GEMM launches of one epoch (fwd 100->256, fwd 256->256, dgrad, wgrad)
OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:'k_tc_gemm' -s 140 -c 12 \
    -o $OUT/prof_gemm_r1g python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_r1g.log 2>&1
