#!/bin/bash
# r1h: launch list of one measured epoch (after 3 warm-up epochs)
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 1800 -c 620 --csv \
    --log-file $OUT/launches_r1h.csv python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_bench_r1h.log 2>&1
