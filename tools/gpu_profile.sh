#!/bin/bash
# Round-2 evidence run: all GPU tests, smoke, the default bench line, the
# ncu launch list of the same command, and ncu --set full captures of the
# three block kernels (cold = ncu's cache flush per replay; warm =
# --cache-control none inside the running block loop).
TAG=${1:-r2prof}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi -L > $O/smi.txt 2>&1
timeout 2000 python -m pytest tests/ -q -m gpu --durations=40 -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
cp gpurun_out/sanitizer_*.log $O/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-paced --no-max-rt --no-c5 > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(k_back|k_front|k_reduce)$' -s 30 -c 3 \
   -o $O/prof python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-paced --no-max-rt --no-c5 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:'^(k_back|k_front|k_reduce)$' -s 90 -c 3 \
   -o $O/warm python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-paced --no-max-rt --no-c5 > $O/ncu_warm.log 2>&1
for f in $O/*.log; do echo "== $f"; tail -n 3 $f; done
tail -c 800 $O/bench.json
