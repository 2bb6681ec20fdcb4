# A/B helper: bash profiles/ab.sh "ENV=a" "ENV=b" ...  (runs gpu tests first, then bench per env)
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 | tee gpurun_out/ab_tests.log
i=0
for cfg in "$@"; do i=$((i+1))
  env $cfg timeout 300 python bench.py --steps ${STEPS:-3} --no-cpu > gpurun_out/ab_$i.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$i.log').read().strip().splitlines()[-1]); k=d['kernels_ms_per_epoch']; print('$cfg', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']*1e3,1), {a:round(b,2) for a,b in k.items()}, d['last_epoch']['train_loss'])" || tail -5 gpurun_out/ab_$i.log
done
