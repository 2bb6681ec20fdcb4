#!/bin/bash
# plan adoption re-uploads without device-wide syncs: adaptive / multirank / setup GPU tests,
# then the re-solve phase breakdown at the bench config (two passes)
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_multirank.py tests/test_gpu_setup.py tests/test_gpu_baseline_configs.py tests/test_gpu_fused.py -q > $O/gputest_r2q.log 2>&1; echo "rc $?" >> $O/gputest_r2q.log
for i in 1 2; do
QGNN_RESOLVE_PROFILE=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > $O/resolve_r2q_$i.log 2>&1
done
