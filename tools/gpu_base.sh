#!/bin/bash
# Baseline check: GPU tests, smoke, default bench line.
TAG=${1:-base}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi -L > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests/ -x -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
for f in $O/*.log; do tail -n 3 $f; done
tail -c 600 $O/bench.json
