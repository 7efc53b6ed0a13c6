#!/bin/bash
O=gpurun_out/r2v
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_auralizer.py tests/test_gpu_convolver.py tests/test_gpu_sanitizer.py tests/test_gpu_shard.py tests/test_gpu_dropin_cpp.py -q -s -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cp gpurun_out/sanitizer_*.log $O/ 2>/dev/null
grep -E "paced|passed|failed|Error" $O/pytest.log | head -20; tail -3 $O/pytest.log
