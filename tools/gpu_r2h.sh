#!/bin/bash
O=gpurun_out/r2h
mkdir -p $O
timeout 600 python tools/exp_cycle.py c3 > $O/exp_cycle_c3.json 2> $O/exp_cycle_c3.err
timeout 900 python bench.py --steps 500 --warmup 20 --no-max-rt --no-c5 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --gpus 2 --steps 50 --warmup 5 --no-max-rt > $O/bench2.json 2> $O/bench2.err
timeout 600 python -m pytest tests/test_gpu_auralizer.py tests/test_gpu_convolver.py tests/test_gpu_engine.py tests/test_gpu_shard.py -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cut -c1-1500 $O/exp_cycle_c3.json; tail -2 $O/exp_cycle_c3.err; tail -c 1200 $O/bench.json; tail -3 $O/bench.err; tail -c 3000 $O/bench2.json; grep -v "^\[rank\|^W\|^\*" $O/bench2.err | tail -5; tail -3 $O/pytest.log
