for v in 0 1 2 3 0; do
  if [ $v = 0 ]; then L=""; else L=$PWD/paper_2306_01381_b200/_lib/l2v$v/libqgnn_b200.so; fi
  QGNN_LIB=$L timeout 400 python bench.py --steps 10 --no-cpu > gpurun_out/ab_l2_$v.log 2>&1
  echo "v=$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_l2_$v.log) $(grep -o '"spmm_fwd": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_l2_$v.log) $(grep -o '"spmm_bwd": {"ms_per_epoch": [0-9.]*' gpurun_out/ab_l2_$v.log)" >> gpurun_out/ab_l2.txt
done
