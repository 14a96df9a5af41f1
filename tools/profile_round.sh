#!/bin/bash
# Round measurement batch on one B200 (run under gpurun from the repo root).
# Every command runs plain first; ncu passes only after it exited 0.
# Outputs land in gpurun_out/ (scratch); summaries are copied to profiles/.
set -u
R=${1:-r01d}
O=gpurun_out
python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err || exit 1
python tools/bench_diag.py 3 > $O/${R}_diag.json 2>&1 || exit 1
for mode in f64 f32 diag; do
  python tools/profile_loop.py C1-image-like 400 $mode > $O/${R}_loop_$mode.txt 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k regex:k_rbd_persistent --launch-skip 1 -c 1 \
      -f -o $O/${R}_prof_$mode python tools/profile_loop.py C1-image-like 400 $mode > $O/${R}_ncu_$mode.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/${R}_ncu_bench.log 2>&1
echo done
