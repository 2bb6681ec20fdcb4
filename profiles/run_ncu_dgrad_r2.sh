#!/bin/bash
# --set full of the input-gradient GEMMs: layer-3 (K = 48 -> N = 256, ReLU-masked epilogue;
# the 33rd k_tc_gemm launch of an epoch) and layer-2 (256 -> 256 masked; the 57th)
O=gpurun_out
for spec in "32:l3" "56:l2"; do
  skip=${spec%%:*}; tag=${spec##*:}
  QGNN_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm \
      -s $skip -c 1 -o $O/prof_dgrad_${tag}_r2 python bench.py --steps 1 --warmup 1 --no-cpu \
      > $O/ncu_dgrad_${tag}_r2.log 2>&1
done
