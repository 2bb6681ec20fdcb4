timeout 300 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/md_test.log 2>&1; echo "rc $?" >> gpurun_out/md_test.log
for v in 0 1 0 1; do
  QGNN_ONE_DGRAD=$v timeout 400 python bench.py --steps 10 --no-cpu > gpurun_out/ab_md_$v.log 2>&1
  echo "v=$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_md_$v.log) $(grep -o '"gemm_dgrad": {"ms_per_epoch": [0-9.]*, "launches_per_epoch": [0-9.]*' gpurun_out/ab_md_$v.log)" >> gpurun_out/ab_md.txt
done
