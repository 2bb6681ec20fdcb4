#!/bin/bash
# r1i: launch list of one measured epoch with DRAM traffic per launch (-> ncu_traffic.json),
# and --set full of the top SpMM launches (fwd 256-wide, fwd grouped 100-wide).
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_' -s 1650 -c 560 --csv --log-file $OUT/traffic_r1i.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_traffic_r1i.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_spmm_f32" -s 24 -c 3 \
    -o $OUT/prof_spmm_r1i python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_spmm_r1i.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_quantize_pack_f32" -s 10 -c 1 \
    -o $OUT/prof_k1_r1i python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_k1_r1i.log 2>&1
