#!/bin/bash
# k_spmm_wide: L1 prefetch of the epilogue's self row / mask word at row start
# (QGNN_LIB = a -DQGNN_SPMM_PF build) vs the default build
O=gpurun_out
for v in 0 1 0 1 0 1; do
  if [ $v = 1 ]; then export QGNN_LIB=$PWD/paper_2306_01381_b200/_lib_pf/libqgnn_b200.so; else unset QGNN_LIB; fi
  timeout 400 python bench.py --steps 10 --no-cpu > $O/ab_spf_$v.log 2>&1
  echo "pf=$v $(grep -o '"ms_per_step": [0-9.]*' $O/ab_spf_$v.log) $(grep -o '"spmm_fwd": {"ms_per_epoch": [0-9.]*' $O/ab_spf_$v.log) $(grep -o '"spmm_bwd": {"ms_per_epoch": [0-9.]*' $O/ab_spf_$v.log) $(grep -o '"sm_mhz": [0-9.]*' $O/ab_spf_$v.log)" >> $O/ab_spmm_pf.txt
done
