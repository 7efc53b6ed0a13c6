#!/bin/bash
O=gpurun_out/r2o
mkdir -p $O
timeout 600 python tools/exp_cycle.py c3 > $O/exp_cycle_c3.json 2> $O/exp_cycle_c3.err
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:'^k_back' -s 40 -c 1 -o $O/c2_back_warm \
   python bench.py --config c2 --steps 60 --warmup 3 --no-cpu-baseline --no-paced --no-max-rt --no-c5 > $O/ncu_c2_warm.log 2>&1
bash tools/gpu_sweep.sh r2sweep2
head -c 400 $O/exp_cycle_c3.json; tail -2 $O/ncu_c2_warm.log
