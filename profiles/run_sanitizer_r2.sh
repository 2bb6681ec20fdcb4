#!/bin/bash
# compute-sanitizer over the kernel unit tests: memcheck on the
# codec / SpMM-variant / dense tests, racecheck + synccheck on the shared-memory
# kernels (tcgen05 GEMM with 2-CTA multicast, SpMM hub finish, K1/K3).
# Output: gpurun_out/sanitizer_*.log (summarised into profiles/sanitizer_r2.txt).
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out
mkdir -p $O
run() {  # tool, log, pytest selection...
  local tool=$1 log=$2; shift 2
  timeout 1500 $CS --tool $tool --target-processes all --error-exitcode 99 \
      python -m pytest -q -p no:cacheprovider "$@" > $O/$log 2>&1
  echo "$tool $log rc=$?" >> $O/sanitizer_rc.txt
}
rm -f $O/sanitizer_rc.txt
run memcheck sanitizer_memcheck_codec.log tests/test_gpu_codec.py
run memcheck sanitizer_memcheck_spmm.log tests/test_gpu_spmm_variants.py -k "default_dispatch or relu_mask or subrange"
run memcheck sanitizer_memcheck_ops.log tests/test_gpu_ops.py
run racecheck sanitizer_racecheck_ops.log tests/test_gpu_ops.py -k "dense_f32"
run racecheck sanitizer_racecheck_spmm.log tests/test_gpu_spmm_variants.py -k "default_dispatch and (47 or 100 or 256)"
run synccheck sanitizer_synccheck_ops.log tests/test_gpu_ops.py -k "dense_f32"
run initcheck sanitizer_initcheck_codec.log tests/test_gpu_codec.py -k "random_sets_f32 or scatter"
cat $O/sanitizer_rc.txt
