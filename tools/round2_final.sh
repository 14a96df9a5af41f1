#!/bin/bash
# Round-2 final measurement batch on one B200 (run under gpurun from the repo root):
# the default bench line, the reference arm, the bench launch list and one
# ncu --set full capture of the headline loop kernel. Each command runs plain
# first; ncu passes only after it exited 0.
set -u
R=${1:-r02z}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/${R}_smi.txt
python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err || { echo bench failed; exit 1; }
python bench.py --impl reference > $O/${R}_bench_ref.json 2> $O/${R}_bench_ref.err || { echo ref failed; exit 1; }
python tools/profile_loop.py C2-tall - f64 > $O/${R}_loop_c2.txt 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary > $O/${R}_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rbd_persistent --launch-skip 1 -c 1 \
    -f -o $O/${R}_prof_c2 python tools/profile_loop.py C2-tall - f64 > $O/${R}_ncu_c2.log 2>&1
echo done
