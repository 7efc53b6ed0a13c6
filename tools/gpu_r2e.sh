#!/bin/bash
O=gpurun_out/r2e
mkdir -p $O
timeout 600 python tools/exp_cycle.py c3 > $O/exp_cycle.json 2> $O/exp_cycle.err
timeout 900 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_engine.py tests/test_gpu_shard.py tests/test_gpu_auralizer.py tests/test_gpu_convolver.py -q -s -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
cp gpurun_out/sanitizer_*.log $O/ 2>/dev/null
# racecheck of k_back alone, for the record (mbarrier/TMA false positives)
timeout 600 compute-sanitizer --tool racecheck --kernel-name regex:k_back -c 4 --log-file $O/racecheck_k_back.log python tests/sanitize_workload.py > /dev/null 2>&1
timeout 900 python tools/exp_l2.py c2 > $O/exp_l2_c2.jsonl 2> $O/exp_l2.err
cat $O/exp_cycle.json; tail -3 $O/exp_cycle.err; tail -5 $O/pytest_gpu.log; tail -3 $O/racecheck_k_back.log; cut -c1-600 $O/exp_l2_c2.jsonl; tail -3 $O/exp_l2.err
