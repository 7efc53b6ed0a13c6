#!/bin/bash
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_engine.py tests/test_gpu_shard.py tests/test_gpu_auralizer.py tests/test_gpu_convolver.py tests/test_gpu_fullsize.py tests/test_gpu_dropin_cpp.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
cp gpurun_out/sanitizer_*.log $O/ 2>/dev/null
timeout 600 compute-sanitizer --tool racecheck --kernel-name kns=k_backILi -c 4 --log-file $O/racecheck_k_back.log python tests/sanitize_workload.py > /dev/null 2>&1
timeout 600 python tools/exp_cycle.py c3 > $O/exp_cycle.json 2> $O/exp_cycle.err
timeout 300 python -c "
import sys; sys.argv=['x','c2']; sys.path.insert(0,'tools'); import exp_l2, json; print(json.dumps(exp_l2.run('c2')))" > $O/exp_l2_c2.json 2> $O/exp_l2.err
tail -5 $O/pytest_gpu.log; tail -3 $O/racecheck_k_back.log; head -c 700 $O/exp_cycle.json; echo; head -c 900 $O/exp_l2_c2.json; tail -3 $O/exp_l2.err
