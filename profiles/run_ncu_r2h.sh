#!/bin/bash
# r2h (end of round 2: mask bits, chunk words, merged input gradients, batched host copies):
# a launch list with DRAM traffic per launch over >= 2 eager epochs (last complete one ->
# ncu_traffic.json), the gpu__time_duration-only launch list (the profiling recipe's pass),
# and --set full of one launch each of the top kernels.
OUT=gpurun_out
QGNN_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'k_' -s 1000 -c 1500 --csv --log-file $OUT/traffic_r2h.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_traffic_r2h.log 2>&1
QGNN_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1000 -c 400 \
    --csv --log-file $OUT/launches_r2h.csv python bench.py --steps 1 --warmup 3 --no-cpu \
    > $OUT/ncu_launches_r2h.log 2>&1
for spec in "k_spmm_wide:1" "k_spmm_f32g2:0" "k_spmm_sorted:0" "k_tc_gemm:2" "k_quantize_pack_grp:2" "k_dequant_rows_f32:0"; do
  k=${spec%%:*}; skip=${spec##*:}
  QGNN_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" \
      -s $skip -c 1 -o $OUT/prof_${k}_r2h python bench.py --steps 1 --warmup 1 --no-cpu \
      > $OUT/ncu_${k}_r2h.log 2>&1
done
