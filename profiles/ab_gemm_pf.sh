# tcgen05 GEMM A/B: cta_group::1 (PAIR=0) vs CTA pair (PAIR=1), A prefetched into L2 PF chunks ahead
for pair in 0 1; do for pf in 0 4 8 16 32; do
  QGNN_GEMM_PAIR=$pair QGNN_GEMM_PF=$pf DBG=0 CLUSTERS=2 SHAPES=100x256,256x256,256x48,48x256 \
    timeout 180 python profiles/gemm_micro.py 2>&1 | sed "s/^/pair=$pair pf=$pf /" >> gpurun_out/ab_gemm_pf.txt
done; done
