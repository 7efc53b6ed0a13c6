#!/bin/bash
O=gpurun_out/r2d
mkdir -p $O
timeout 2000 python -m pytest tests/ -q -s -m gpu --durations=30 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
cp gpurun_out/sanitizer_*.log $O/ 2>/dev/null
timeout 600 python tools/exp_cycle.py c3 > $O/exp_cycle.json 2> $O/exp_cycle.err
timeout 900 python bench.py --steps 200 --warmup 20 > $O/bench.json 2> $O/bench.err
grep -E "^(c1|c3|c4|c5|delta)|passed|failed|FAILED" $O/pytest_gpu.log | head -60; cat $O/exp_cycle.json; tail -3 $O/exp_cycle.err; tail -c 1500 $O/bench.json; tail -5 $O/bench.err
