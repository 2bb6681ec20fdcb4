#!/bin/bash
# r1f: launch list of one measured epoch (after 3 warm-up epochs, ~620 launches each)
# and --set full captures of the top SpMM and K1 launches; plus the gather probe.
OUT=gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a profiles/gather_probe.cu -o $OUT/gather_probe && \
  $OUT/gather_probe > $OUT/gather_probe_r1f.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 1900 -c 700 --csv \
    --log-file $OUT/launches_r1f.csv python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_bench_r1f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_spmm_f32' -s 60 -c 6 \
    -o $OUT/prof_spmm_r1f python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_spmm_r1f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_quantize_pack_f32' -s 40 -c 3 \
    -o $OUT/prof_k1_r1f python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_k1_r1f.log 2>&1
