#!/bin/bash
# GPU call: bench lines for every BASELINE config and the c4 block-size
# sweep (the c3 line carries the max real-time search and the c5 line).
# usage: bash tools/gpu_sweep.sh TAG
TAG=${1:-sweep}
O=gpurun_out/$TAG
mkdir -p $O
B="timeout 900 python bench.py --warmup 10 --no-paced --no-max-rt --no-c5"
$B --config c1 --steps 2000 > $O/c1.json 2> $O/c1.err
$B --config c2 --steps 2000 > $O/c2.json 2> $O/c2.err
for N in 32 64 128 256 512 1024; do
  CPU="--no-cpu-baseline"; if [ $N = 64 ] || [ $N = 1024 ]; then CPU="--cpu-blocks 3"; fi
  $B --config c4 --block $N --steps 500 $CPU > $O/c4_n$N.json 2> $O/c4_n$N.err
done
$B --config c5 --steps 300 --cpu-blocks 3 > $O/c5.json 2> $O/c5.err
timeout 900 python bench.py --steps 2000 --warmup 20 > $O/c3.json 2> $O/c3.err
for f in $O/*.err; do tail -n 2 $f; done
