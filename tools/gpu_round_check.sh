set -u
O=gpurun_out; R=r02h
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/${R}_smi.txt
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $O/${R}_gputests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err; echo "bench rc=$?"
tail -3 $O/${R}_gputests.log
