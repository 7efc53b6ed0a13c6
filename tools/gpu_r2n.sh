#!/bin/bash
# After the host split: all GPU tests, the per-config bench lines, the c2
# k_back ncu capture (L2-resident roofline), the Section VI sweep CSVs.
O=gpurun_out/r2n
mkdir -p $O
timeout 2000 python -m pytest tests/ -q -m gpu --durations=40 -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
cp gpurun_out/sanitizer_*.log $O/ 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^k_back' -s 10 -c 1 -o $O/c2_back \
   python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline --no-paced --no-max-rt --no-c5 > $O/ncu_c2.log 2>&1
bash tools/gpu_sweep.sh r2sweep
bash tools/gpu_sweeps_csv.sh r2csv
tail -4 $O/pytest_gpu.log; tail -3 $O/ncu_c2.log
