#!/bin/bash
OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:'k_quantize_pack_f32' -s 40 -c 2 \
    -o $OUT/prof_k1_r1d python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_r1d_a.log 2>&1
