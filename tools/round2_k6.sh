#!/bin/bash
# K6 CTA-pair kernel: parity tests, then device timing of the C4 batch for both kernels.
set -u
O=gpurun_out; R=${1:-r02k6}
mkdir -p $O
( timeout 600 python -m pytest tests/test_gpu_project_f32.py -m gpu -x -q ) > $O/${R}_tests.log 2>&1; echo "tests rc=$?"; tail -15 $O/${R}_tests.log
for p in 0 1; do for sk in 1 2 4; do
  RBD_K6_PAIR=$p RBD_K6_SPLITK=$sk timeout 300 python tools/time_k6.py 2>&1 | tail -3
done; done > $O/${R}_time.txt 2>&1; cat $O/${R}_time.txt
