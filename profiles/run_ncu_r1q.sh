#!/bin/bash
# r1q (final, end of round 1): gpu tests, smoke, the default bench line, a launch list with DRAM
# traffic per launch over >= 2 eager epochs (last complete one -> ncu_traffic.json), and
# --set full of one launch each of the top kernels: 256-wide SpMM, degree-sorted narrow
# SpMM, grouped 100-wide SpMM, the K-major GEMM and K1.
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests_r1q.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke_r1q.log 2>&1
timeout 600 python bench.py > $OUT/bench_r1q.log 2>&1
QGNN_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'k_' -s 1000 -c 1500 --csv --log-file $OUT/traffic_r1q.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_traffic_r1q.log 2>&1
for spec in "k_spmm_wide:0" "k_spmm_sorted:0" "k_spmm_f32g2:0" "k_tc_gemm:2" "k_quantize_pack_lean:2"; do
  k=${spec%%:*}; skip=${spec##*:}
  QGNN_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" \
      -s $skip -c 1 -o $OUT/prof_${k}_r1q python bench.py --steps 1 --warmup 1 --no-cpu \
      > $OUT/ncu_${k}_r1q.log 2>&1
done
