#!/bin/bash
# GPU call: bandwidth probe + ncu capture of k_back on c3.
TAG=${1:-probe}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 tools/_bw_probe > $O/bw_probe.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_back$|k_back<' -s 10 -c 2 \
   -o $O/prof python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-paced > $O/ncu_full.log 2>&1
tail -n 3 $O/ncu_full.log
