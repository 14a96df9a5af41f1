#!/bin/bash
# HEAD check + final measurement batch on one B200 (run under gpurun from the repo root):
# GPU tests, smoke(), then tools/round2_final.sh (bench, reference arm, launch list, ncu).
set -u
R=${1:-r02y}
O=gpurun_out
mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $O/${R}_gputests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 $O/${R}_gputests.log; tail -1 $O/${R}_smoke.log
bash tools/round2_final.sh $R
