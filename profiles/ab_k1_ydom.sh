#!/bin/bash
# K1 element decision: x-domain (QGNN_K1_YDOM=0) vs y-domain floor(x + 1 - u) (=1):
# codec/engine parity tests, wire digests and speed of the microbenchmark, bench A/B
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_engine.py tests/test_gpu_baseline_configs.py tests/test_gpu_fused.py -x -q > $O/k1yd_test.log 2>&1; echo "rc $?" >> $O/k1yd_test.log
for y in 0 1; do QGNN_K1_YDOM=$y timeout 300 python profiles/k1_bench.py 400000 2>&1 | sed "s/^/ydom=$y /" >> $O/ab_k1_ydom.txt; done
for y in 0 1 0 1 0 1; do
  QGNN_K1_YDOM=$y timeout 400 python bench.py --steps 10 --no-cpu > $O/ab_k1y_$y.log 2>&1
  echo "ydom=$y $(grep -o '"ms_per_step": [0-9.]*' $O/ab_k1y_$y.log) $(grep -o '"quant": {"ms_per_epoch": [0-9.]*' $O/ab_k1y_$y.log) $(grep -o '"sm_mhz": [0-9.]*' $O/ab_k1y_$y.log)" >> $O/ab_k1_ydom.txt
done
