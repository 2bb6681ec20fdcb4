#!/bin/bash
# grouped-lane forward K3 (default build) — GPU tests; then the backward scatter-add at
# 24 CTAs/SM (QGNN_LIB = a -DQGNN_K3B_MINB=24 build, 38 registers) vs the default
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $O/k3fwd_test.log 2>&1; echo "rc $?" >> $O/k3fwd_test.log
for v in 0 1 0 1 0 1; do
  if [ $v = 1 ]; then export QGNN_LIB=$PWD/paper_2306_01381_b200/_lib_b/libqgnn_b200.so; else unset QGNN_LIB; fi
  timeout 400 python bench.py --steps 10 --no-cpu > $O/ab_k3o_$v.log 2>&1
  echo "minb24=$v $(grep -o '"ms_per_step": [0-9.]*' $O/ab_k3o_$v.log) $(grep -o '"dequant": {"ms_per_epoch": [0-9.]*' $O/ab_k3o_$v.log) $(grep -o '"sm_mhz": [0-9.]*' $O/ab_k3o_$v.log)" >> $O/ab_k3_occ.txt
done
