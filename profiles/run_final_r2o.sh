#!/bin/bash
# r2o: GPU tests, smoke and the default bench line of the final round-2 tree
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest_r2o.log 2>&1; echo "rc $?" >> $O/gputest_r2o.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r2o.log 2>&1
timeout 900 python bench.py > $O/bench_r2o.log 2>&1
