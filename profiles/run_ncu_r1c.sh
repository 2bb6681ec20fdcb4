#!/bin/bash
OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:'k_spmm_f32<2>|k_spmm_f32' -s 250 -c 3 \
    -o $OUT/prof_spmm256_r1c python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_r1c_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_quantize_pack_f32|k_dequant_f32' -s 40 -c 4 \
    -o $OUT/prof_codec_r1c python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_r1c_b.log 2>&1
