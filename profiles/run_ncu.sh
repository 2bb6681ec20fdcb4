#!/bin/bash
# ncu evidence for the bench workload (run under gpurun on ONE GPU).
#   launches: every kernel launch of 1 measured epoch after warm-up (cold-cache, serialised)
#   full:     --set full capture of the top kernels
set -x
TAG=${1:-r1}
OUT=gpurun_out
# warm-up epochs launch ~440 kernels each; skip 3 epochs, capture 1 epoch
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 1330 -c 450 --csv \
    --log-file $OUT/launches_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_bench_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_csr_aggregate|k_sgemm|k_quantize_pack|k_dequant_scatter' \
    -s 1330 -c 12 -o $OUT/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_full_${TAG}.log 2>&1
ls -la $OUT
