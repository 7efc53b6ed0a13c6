#!/bin/bash
# GPU call: gpu tests + one bench line (no profiler). usage: bash tools/gpu_quick.sh TAG [bench args...]
TAG=${1:-quick}; shift
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/ -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py "$@" > $O/bench.json 2> $O/bench.err
tail -n 3 $O/pytest_gpu.log; tail -n 3 $O/bench.err
