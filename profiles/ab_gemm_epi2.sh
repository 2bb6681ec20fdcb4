timeout 300 python -m pytest tests/test_gpu_ops.py -x -q -k dense > gpurun_out/epi2_test.log 2>&1; echo "rc $?" >> gpurun_out/epi2_test.log
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_baseline_configs.py -x -q >> gpurun_out/epi2_test.log 2>&1; echo "rc $?" >> gpurun_out/epi2_test.log
for e in 0 1; do QGNN_GEMM_EPI2=$e DBG=0 CLUSTERS=2 SHAPES=48x256,100x256,256x256,256x48 timeout 180 python profiles/gemm_micro.py 2>&1 | sed "s/^/epi2=$e /" >> gpurun_out/ab_epi2.txt; done
for e in 0 1 0 1 0 1; do
  QGNN_GEMM_EPI2=$e timeout 400 python bench.py --steps 10 --no-cpu > gpurun_out/ab_e2_$e.log 2>&1
  echo "epi2=$e $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_e2_$e.log) $(grep -o '"gemm_fwd": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_e2_$e.log) $(grep -o '"gemm_dgrad": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_e2_$e.log)" >> gpurun_out/ab_epi2.txt
done
