#!/bin/bash
# r2l: GPU tests with the weight-gradient conv2 GEMM, smoke, the default bench line,
# and one bench pass with the re-solve phase breakdown
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest_r2l.log 2>&1; echo "rc $?" >> $O/gputest_r2l.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r2l.log 2>&1
timeout 900 python bench.py > $O/bench_r2l.log 2>&1
QGNN_RESOLVE_PROFILE=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > $O/resolve_r2l.log 2>&1
