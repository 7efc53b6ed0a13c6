#!/bin/bash
# GPU call: shard + drop-in tests, 2-process sharded bench on one GPU, max real-time search.
TAG=${1:-shard}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_dropin_cpp.py -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for t in test_convolver test_auralizer test_oracle; do timeout 600 tests/cpp/_bin/$t > $O/cpp_$t.log 2>&1; echo "rc=$?" >> $O/cpp_$t.log; done
timeout 1200 tests/cpp/_bin/acceptance > $O/cpp_acceptance.log 2>&1; echo "rc=$?" >> $O/cpp_acceptance.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus 2 --steps 500 --warmup 10 > $O/bench_g2.json 2> $O/bench_g2.err
timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-paced --max-rt > $O/bench_maxrt.json 2> $O/bench_maxrt.err
for f in $O/*.log; do tail -n 2 $f; done
