# A/B of the GEMM stream (QGNN_GEMM_STREAM): bench device ms/epoch per setting
timeout 300 python -m pytest tests/test_gpu_engine.py -q -k "gemm_stream or side_stream or merged" > gpurun_out/gs_test.log 2>&1
for v in 0 1 2 0 1 2; do
  QGNN_GEMM_STREAM=$v timeout 400 python bench.py --steps 10 --no-cpu > gpurun_out/ab_gs_$v.log 2>&1
  echo "gs=$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_gs_$v.log) $(grep -o '"median_ms_per_step": [0-9.]*' gpurun_out/ab_gs_$v.log)" >> gpurun_out/ab_gs.txt
done
