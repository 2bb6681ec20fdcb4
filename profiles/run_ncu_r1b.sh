#!/bin/bash
# Per-kernel ncu --set full captures of the current top kernels (1 GPU).
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 1500 -c 520 --csv \
    --log-file $OUT/launches_r1b.csv python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_bench_r1b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_spmm_f32' -s 240 -c 6 \
    -o $OUT/prof_spmm_r1b python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_spmm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_quantize_pack|k_tc_gemm|k_relu_backward|k_dequant' -s 120 -c 8 \
    -o $OUT/prof_misc_r1b python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_misc.log 2>&1
