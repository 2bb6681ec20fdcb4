#!/bin/bash
# forward K3 (k_dequant_f32): G lanes per message + header/payload together (default build)
# vs one warp per message (QGNN_LIB = the same tree with the previous kernel); both with the
# backward scatter-add at 24 CTAs/SM
O=gpurun_out
for v in 0 1 0 1 0 1; do
  if [ $v = 0 ]; then export QGNN_LIB=$PWD/paper_2306_01381_b200/_lib_c/libqgnn_b200.so; else unset QGNN_LIB; fi
  timeout 400 python bench.py --steps 10 --no-cpu > $O/ab_k3f_$v.log 2>&1
  echo "grouped=$v $(grep -o '"ms_per_step": [0-9.]*' $O/ab_k3f_$v.log) $(grep -o '"dequant": {"ms_per_epoch": [0-9.]*' $O/ab_k3f_$v.log) $(grep -o '"sm_mhz": [0-9.]*' $O/ab_k3f_$v.log)" >> $O/ab_k3_fwd_grp.txt
done
