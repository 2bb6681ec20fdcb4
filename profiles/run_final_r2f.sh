#!/bin/bash
# r2f (end of round 2): GPU tests, smoke, the default bench line and the reference arm
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest_r2f.log 2>&1; echo "rc $?" >> $O/gputest_r2f.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r2f.log 2>&1
timeout 900 python bench.py > $O/bench_r2f.log 2>&1
timeout 1200 python bench.py --impl reference --steps 2 > $O/bench_r2f_reference.log 2>&1
