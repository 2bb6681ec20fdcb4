timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_multirank.py tests/test_gpu_baseline_configs.py tests/test_gpu_chain.py -x -q > gpurun_out/host_test.log 2>&1; echo "rc $?" >> gpurun_out/host_test.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --no-cpu > gpurun_out/bench_host$i.log 2>&1
grep '^{' gpurun_out/bench_host$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('dev', d['ms_per_step'], 'wall', d['wall_s_per_step']*1e3, 'e2e', d['e2e']['value']*1e3, 'e2e_dev', d['e2e']['device_ms_per_step'])" >> gpurun_out/host_ab.txt
done
