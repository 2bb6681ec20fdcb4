timeout 300 python -m pytest tests/test_gpu_engine.py tests/test_gpu_ops.py tests/test_gpu_baseline_configs.py -x -q > gpurun_out/mb_test.log 2>&1; echo "rc $?" >> gpurun_out/mb_test.log
for b in 0 1 0 1 0 1; do
  QGNN_MASK_BITS=$b timeout 400 python bench.py --steps 10 --no-cpu > gpurun_out/ab_mb_$b.log 2>&1
  echo "bits=$b $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_mb_$b.log) $(grep -o '"gemm_dgrad": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_mb_$b.log) $(grep -o '"gemm_fwd": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_mb_$b.log)" >> gpurun_out/ab_mask_bits.txt
done
