#!/bin/bash
# All GPU tests (no -x) with durations; the c3 full-size NLMS delta study.
O=gpurun_out/r2c
mkdir -p $O
timeout 1800 python -m pytest tests/ -q -m gpu --durations=30 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python tools/nlms_delta.py c3 > $O/nlms_delta_c3.jsonl 2> $O/nlms_delta_c3.err
tail -n 45 $O/pytest_gpu.log; cat $O/nlms_delta_c3.jsonl | cut -c1-400; tail -3 $O/nlms_delta_c3.err
