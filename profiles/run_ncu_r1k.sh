#!/bin/bash
# r1k (end of session 2): launch list of one measured epoch (eager, kstats off -> graph replay
# is not profiled per kernel by ncu launch lists; QGNN_GRAPH=0 keeps one launch per kernel),
# DRAM traffic per class, and --set full of the top SpMM, GEMM and K1 launches.
OUT=gpurun_out
QGNN_GRAPH=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'k_' -s 1650 -c 560 --csv --log-file $OUT/traffic_r1k.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_traffic_r1k.log 2>&1
QGNN_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:'k_spmm_f32|k_tc_gemm|k_quantize_pack_lean' \
    -s 20 -c 6 -o $OUT/prof_top_r1k python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_top_r1k.log 2>&1
