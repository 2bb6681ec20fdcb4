#!/bin/bash
# r2m: frontier knapsack tables + radix grouping + setup-time window buffer:
# GPU tests, then the re-solve phase breakdown at the bench config (two passes)
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest_r2m.log 2>&1; echo "rc $?" >> $O/gputest_r2m.log
for i in 1 2; do
QGNN_RESOLVE_PROFILE=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > $O/resolve_r2m_$i.log 2>&1
done
