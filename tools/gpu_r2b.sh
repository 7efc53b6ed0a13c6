#!/bin/bash
# GPU tests (with durations), smoke, default bench; host facts.
TAG=${1:-r2b}
O=gpurun_out/$TAG
mkdir -p $O
nproc > $O/host.txt; free -g >> $O/host.txt; lscpu | head -20 >> $O/host.txt
timeout 1500 python -m pytest tests/ -q -m gpu --durations=25 -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
tail -n 40 $O/pytest_gpu.log; tail -3 $O/smoke.log; tail -c 400 $O/bench.json
