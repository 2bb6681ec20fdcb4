#!/bin/bash
# grouped K1 (y-domain) occupancy: 32 elements/lane at 3 CTAs/SM (default), 16 elements/lane
# at 4 CTAs/SM (QGNN_K1_EPL=16), 32 elements/lane at 4 CTAs/SM (64 registers, spills; QGNN_LIB build)
O=gpurun_out
timeout 300 python profiles/k1_bench.py 400000 2>&1 | sed "s/^/epl32x3 /" >> $O/ab_k1_occ.txt
QGNN_K1_EPL=16 timeout 300 python profiles/k1_bench.py 400000 2>&1 | sed "s/^/epl16x4 /" >> $O/ab_k1_occ.txt
QGNN_LIB=$PWD/paper_2306_01381_b200/_lib_k1/libqgnn_b200.so timeout 300 python profiles/k1_bench.py 400000 2>&1 | sed "s/^/epl32x4 /" >> $O/ab_k1_occ.txt
