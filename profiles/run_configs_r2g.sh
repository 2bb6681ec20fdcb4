#!/bin/bash
# r2g: bench lines of BASELINE configs 2, 3, 5 and config 4 at fixed 4 / 2 bits with the final round-2 code
O=gpurun_out
for c in 2 3 5; do timeout 900 python bench.py --config $c > $O/bench_r2g_cfg$c.log 2>&1; done
for b in 4 2; do timeout 900 python bench.py --bit-mode fixed --bits $b > $O/bench_r2g_cfg4_fixed$b.log 2>&1; done
