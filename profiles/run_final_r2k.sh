#!/bin/bash
# r2k: GPU tests, smoke and the default bench line with the final round-2 code
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest_r2k.log 2>&1; echo "rc $?" >> $O/gputest_r2k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r2k.log 2>&1
timeout 900 python bench.py > $O/bench_r2k.log 2>&1
