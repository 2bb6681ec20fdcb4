#!/bin/bash
# compute-sanitizer over the round-2 additions: GPU-side setup kernels (memcheck,
# racecheck: shared-memory consumer bitmaps) and the packed-halo / engine paths;
# the peer-store transport (memcheck over the loopback group: K1 stores into peer
# arenas, flag signal / wait kernels).
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
run memcheck sanitizer_memcheck_setup.log tests/test_gpu_setup.py -k "not planted or partitions"
run racecheck sanitizer_racecheck_setup.log tests/test_gpu_setup.py -k "partitions_gpu_equal"
run memcheck sanitizer_memcheck_p2p.log tests/test_gpu_multirank.py -k "peer_store_is_bit_identical and 2 and (fixed or adaptive)"
run memcheck sanitizer_memcheck_fused.log tests/test_gpu_fused.py
cat $O/sanitizer_rc.txt
for f in $O/sanitizer_memcheck_setup.log $O/sanitizer_racecheck_setup.log $O/sanitizer_memcheck_p2p.log $O/sanitizer_memcheck_fused.log; do
  echo "== $f"; tail -3 $f; done > $O/sanitizer_r2b_summary.txt
