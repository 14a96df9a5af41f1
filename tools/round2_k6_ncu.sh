#!/bin/bash
# ncu --set full of K6, single-CTA (split 2) and CTA-pair (split 4) kernels on the C4 batch.
set -u
O=gpurun_out; R=${1:-r02k6}
mkdir -p $O
RBD_K6_PAIR=0 RBD_K6_SPLITK=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_project_tf32x3 --launch-skip 1 -c 1 -f -o $O/${R}_prof_single python tools/time_k6.py 2 > $O/${R}_ncu_single.log 2>&1
RBD_K6_PAIR=1 RBD_K6_SPLITK=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_project_tf32x3 --launch-skip 1 -c 1 -f -o $O/${R}_prof_pair python tools/time_k6.py 2 > $O/${R}_ncu_pair.log 2>&1
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv -lms 200 > $O/${R}_smi.txt &
SMI=$!
RBD_K6_PAIR=1 RBD_K6_SPLITK=4 timeout 300 python tools/time_k6.py 300 | tail -3
kill $SMI
sort $O/${R}_smi.txt | uniq -c | sort -rn | head -5
