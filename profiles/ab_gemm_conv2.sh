timeout 300 python -m pytest tests/test_gpu_ops.py -x -q -k dense > gpurun_out/cv2_test.log 2>&1; echo "rc $?" >> gpurun_out/cv2_test.log
for c in 0 1; do QGNN_GEMM_CONV2=$c DBG=0 CLUSTERS=2 SHAPES=256x48,256x256,48x256 timeout 180 python profiles/gemm_micro.py 2>&1 | sed "s/^/conv2=$c /" >> gpurun_out/ab_cv2.txt; done
for c in 0 1 0 1 0 1; do
  QGNN_GEMM_CONV2=$c timeout 400 python bench.py --steps 10 --no-cpu > gpurun_out/ab_c2_$c.log 2>&1
  echo "conv2=$c $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_c2_$c.log) $(grep -o '"gemm_fwd": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_c2_$c.log) $(grep -o '"gemm_wgrad": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_c2_$c.log)" >> gpurun_out/ab_cv2.txt
done
