#!/bin/bash
# K3 backward (k_dequant_rows_f32), then with chunk words per entry: destination row / mask loaded before the message
# chain, header + payload together, 2 chunks per lane for D <= 256
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $O/k3bwd_words_test.log 2>&1; echo "rc $?" >> $O/k3bwd_words_test.log
for i in 1 2; do
  timeout 400 python bench.py --steps 10 --no-cpu > $O/k3bwd_bench_$i.log 2>&1
  echo "run $i $(grep -o '"ms_per_step": [0-9.]*' $O/k3bwd_bench_$i.log) $(grep -o '"dequant": {"ms_per_epoch": [0-9.]*' $O/k3bwd_bench_$i.log) $(grep -o '"quant": {"ms_per_epoch": [0-9.]*' $O/k3bwd_bench_$i.log) $(grep -o '"sm_mhz": [0-9.]*' $O/k3bwd_bench_$i.log)" >> $O/k3bwd_words_r2.txt
done
