#!/bin/bash
# --set full of one K1 launch (D=256, forward layer 1) and one D=100 launch
OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:'k_quantize_pack_f32' -s 7 -c 2 \
    -o $OUT/prof_k1 python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_k1.log 2>&1
