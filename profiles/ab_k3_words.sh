#!/bin/bash
# backward scatter-add: chunk words per entry (QGNN_K3_WORDS=1) vs message -> offset / width (=0)
O=gpurun_out
for w in 0 1 0 1 0 1; do
  QGNN_K3_WORDS=$w timeout 400 python bench.py --steps 10 --no-cpu > $O/ab_k3w_$w.log 2>&1
  echo "k3words=$w $(grep -o '"ms_per_step": [0-9.]*' $O/ab_k3w_$w.log) $(grep -o '"dequant": {"ms_per_epoch": [0-9.]*' $O/ab_k3w_$w.log) $(grep -o '"sm_mhz": [0-9.]*' $O/ab_k3w_$w.log)" >> $O/ab_k3_words.txt
done
