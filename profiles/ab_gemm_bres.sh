# resident-B A/B for the skinny K-major GEMMs (QGNN_GEMM_BRES)
timeout 300 python -m pytest tests/test_gpu_ops.py -x -q -k dense > gpurun_out/bres_test.log 2>&1; echo "rc $?" >> gpurun_out/bres_test.log
for b in 0 1; do
  QGNN_GEMM_BRES=$b DBG=0 CLUSTERS=2 SHAPES=256x48,48x256,100x256,256x256 timeout 180 python profiles/gemm_micro.py 2>&1 | sed "s/^/bres=$b /" >> gpurun_out/ab_gemm_bres.txt
done
for b in 0 1 0 1; do
  QGNN_GEMM_BRES=$b timeout 400 python bench.py --steps 10 --no-cpu > gpurun_out/ab_bres_$b.log 2>&1
  echo "bres=$b $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_bres_$b.log) $(grep -o '"gemm_fwd": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_bres_$b.log) $(grep -o '"gemm_dgrad": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_bres_$b.log)" >> gpurun_out/ab_gemm_bres.txt
done
