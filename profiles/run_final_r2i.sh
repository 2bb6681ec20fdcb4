#!/bin/bash
# r2i (end of round 2): full-size fp32-vs-reference parity on the bench workload, the
# default bench line, smoke
O=gpurun_out
timeout 1500 python profiles/full_parity.py 3 > $O/full_parity_cfg4.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r2i.log 2>&1
timeout 900 python bench.py > $O/bench_r2i.log 2>&1
