#!/bin/bash
# GEMM epilogue ReLU-mask words: loaded once per tile per row and shuffled (default build)
# vs loaded per 32-column block (QGNN_LIB = the previous gemm_tc.cu); dense + engine tests first
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_engine.py tests/test_gpu_chain.py -q > $O/maskrow_test.log 2>&1; echo "rc $?" >> $O/maskrow_test.log
for v in 0 1 0 1 0 1; do
  if [ $v = 0 ]; then export QGNN_LIB=$PWD/paper_2306_01381_b200/_lib_c/libqgnn_b200.so; else unset QGNN_LIB; fi
  timeout 400 python bench.py --steps 10 --no-cpu > $O/ab_mr_$v.log 2>&1
  echo "rowmask=$v $(grep -o '"ms_per_step": [0-9.]*' $O/ab_mr_$v.log) $(grep -o '"gemm_dgrad": {"ms_per_epoch": [0-9.]*' $O/ab_mr_$v.log) $(grep -o '"gemm_fwd": {"ms_per_epoch": [0-9.]*' $O/ab_mr_$v.log) $(grep -o '"sm_mhz": [0-9.]*' $O/ab_mr_$v.log)" >> $O/ab_gemm_maskrow.txt
done
