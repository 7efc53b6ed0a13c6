#!/bin/bash
O=gpurun_out/r2g
mkdir -p $O
for c in c3 c1 c2; do timeout 600 python tools/exp_cycle.py $c > $O/exp_cycle_$c.json 2> $O/exp_cycle_$c.err; done
timeout 900 python bench.py --gpus 2 --steps 50 --warmup 5 --no-max-rt > $O/bench2.json 2> $O/bench2.err
for c in c3 c1 c2; do cat $O/exp_cycle_$c.json | cut -c1-900; tail -2 $O/exp_cycle_$c.err; done
tail -c 2500 $O/bench2.json; tail -20 $O/bench2.err
