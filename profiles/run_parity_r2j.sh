#!/bin/bash
# full-size parity of configs 3 (Yelp-shaped, GraphSAGE) and 2 (Reddit-shaped, 602 features)
timeout 1500 python profiles/full_parity.py 3 3 > gpurun_out/full_parity_cfg3.log 2>&1
free -g > gpurun_out/free.txt
timeout 2400 python profiles/full_parity.py 3 2 > gpurun_out/full_parity_cfg2.log 2>&1
