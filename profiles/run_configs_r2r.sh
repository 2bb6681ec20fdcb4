#!/bin/bash
# r2r: bench lines of BASELINE configs 2, 3, 5 and config 4 at fixed 4 / 2 bits with the end-of-round-2 code (y-domain K1, backward scatter-add chain, re-solve)
O=gpurun_out
for c in 2 3 5; do timeout 900 python bench.py --config $c > $O/bench_r2r_cfg$c.log 2>&1; done
for b in 4 2; do timeout 900 python bench.py --bit-mode fixed --bits $b > $O/bench_r2r_cfg4_fixed$b.log 2>&1; done
