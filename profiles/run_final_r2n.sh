#!/bin/bash
# r2n (end of round 2: y-domain K1, backward scatter-add chain, re-solve): GPU tests,
# smoke, the default bench line; then the launch list with DRAM traffic per launch
# (-> ncu_traffic.json), the time-only launch list, and --set full of one launch each of
# the two kernels changed since r2h.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest_r2n.log 2>&1; echo "rc $?" >> $O/gputest_r2n.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r2n.log 2>&1
timeout 900 python bench.py > $O/bench_r2n.log 2>&1
QGNN_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'k_' -s 1000 -c 1500 --csv --log-file $O/traffic_r2n.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_traffic_r2n.log 2>&1
QGNN_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1000 -c 400 \
    --csv --log-file $O/launches_r2n.csv python bench.py --steps 1 --warmup 3 --no-cpu \
    > $O/ncu_launches_r2n.log 2>&1
for spec in "k_quantize_pack_grp:2" "k_dequant_rows_f32:0"; do
  k=${spec%%:*}; skip=${spec##*:}
  QGNN_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" \
      -s $skip -c 1 -o $O/prof_${k}_r2n python bench.py --steps 1 --warmup 1 --no-cpu \
      > $O/ncu_${k}_r2n.log 2>&1
done
