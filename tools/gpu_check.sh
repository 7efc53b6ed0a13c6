#!/bin/bash
# One gpurun call: GPU tests, smoke, bench line, launch list, ncu capture.
# usage (from repo root, under gpurun): bash tools/gpu_check.sh [tag]
TAG=${1:-check}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi -L > $O/smi.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv >> $O/smi.txt 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-paced > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(k_back|k_front|k_reduce)$' -s 30 -c 3 \
   -o $O/prof python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-paced > $O/ncu_full.log 2>&1
for f in $O/*.log; do tail -n 3 $f; done
