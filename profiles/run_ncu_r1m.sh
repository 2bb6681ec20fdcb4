#!/bin/bash
# r1m (end of session 3): gpu tests, the default bench line, a launch list with DRAM
# traffic per launch over >= 2 eager epochs (the last complete one -> ncu_traffic.json),
# and --set full of the top SpMM (256-wide and narrow), GEMM and K1 launches.
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests_r1m.log 2>&1
timeout 600 python bench.py > $OUT/bench_r1m.log 2>&1
QGNN_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'k_' -s 1000 -c 1500 --csv --log-file $OUT/traffic_r1m.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_traffic_r1m.log 2>&1
QGNN_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_spmm_wide|k_spmm_f32g2|k_tc_gemm|k_quantize_pack_lean' -s 40 -c 8 \
    -o $OUT/prof_top_r1m python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_top_r1m.log 2>&1
