#!/bin/bash
# A/B of the early canceller reduction (AURA_B200_AFC_EARLY) at c3 plus the
# canceller parity tests.
O=gpurun_out/${1:-r3b}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_auralizer.py tests/test_gpu_engine.py -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 1 0 1 0; do
  AURA_B200_AFC_EARLY=$k timeout 300 python tools/exp_back.py --cases nlms >> $O/back_$k.jsonl 2>&1
  AURA_B200_AFC_EARLY=$k timeout 300 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --no-max-rt --no-c5 >> $O/bench_$k.jsonl 2>> $O/bench_$k.err
done
tail -2 $O/pytest.log
