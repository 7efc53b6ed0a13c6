#!/bin/bash
# GPU call: bench lines for every BASELINE config, the c4 block-size sweep
# and the max real-time search (c3 shape). usage: bash tools/gpu_sweep.sh TAG
TAG=${1:-sweep}
O=gpurun_out/$TAG
mkdir -p $O
B="timeout 900 python bench.py --warmup 10 --no-paced"
$B --config c1 --steps 2000 > $O/c1.json 2> $O/c1.err
$B --config c2 --steps 2000 > $O/c2.json 2> $O/c2.err
for N in 32 64 128 256 512 1024; do
  CPU="--no-cpu-baseline"; if [ $N = 64 ] || [ $N = 1024 ]; then CPU="--cpu-blocks 3"; fi
  $B --config c4 --block $N --steps 500 $CPU > $O/c4_n$N.json 2> $O/c4_n$N.err
done
$B --config c5 --steps 300 --cpu-blocks 3 > $O/c5.json 2> $O/c5.err
$B --config c3 --steps 300 --no-cpu-baseline --max-rt > $O/c3_maxrt.json 2> $O/c3_maxrt.err
for f in $O/*.err; do tail -n 2 $f; done
