timeout 300 python -m pytest tests/test_gpu_ops.py -x -q -k dense > gpurun_out/c8_test.log 2>&1; echo "rc $?" >> gpurun_out/c8_test.log
QGNN_GEMM_CLUSTER=8 timeout 300 python -m pytest tests/test_gpu_ops.py -x -q -k dense >> gpurun_out/c8_test.log 2>&1; echo "rc $?" >> gpurun_out/c8_test.log
for c in 2 4 8; do DBG=0 CLUSTERS=$c SHAPES=100x256,256x256,48x256 timeout 180 python profiles/gemm_micro.py >> gpurun_out/c8.txt 2>&1; done
timeout 900 python bench.py --config 2 > gpurun_out/bench_r2g_cfg2b.log 2>&1
