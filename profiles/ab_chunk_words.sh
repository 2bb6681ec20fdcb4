timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_engine.py tests/test_gpu_exchange.py tests/test_gpu_baseline_configs.py tests/test_gpu_multirank.py -x -q > gpurun_out/cw_test.log 2>&1; echo "rc $?" >> gpurun_out/cw_test.log
for v in 0 1 0 1 0 1; do
  QGNN_CHUNK_WORDS=$v timeout 400 python bench.py --steps 10 --no-cpu > gpurun_out/ab_cw_$v.log 2>&1
  echo "v=$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_cw_$v.log) $(grep -o '"spmm_fwd": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_cw_$v.log) $(grep -o '"train_loss": [0-9.]*' gpurun_out/ab_cw_$v.log)" >> gpurun_out/ab_cw.txt
done
