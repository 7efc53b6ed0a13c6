set -x
O=gpurun_out/r2a
mkdir -p $O
BW_L2=1 timeout 300 ./tools/_bw_probe > $O/bw_l2.jsonl 2>&1
timeout 900 python tools/nlms_delta.py > $O/nlms_delta.jsonl 2> $O/nlms_delta.err
nproc > $O/host.txt; lscpu >> $O/host.txt; free -g >> $O/host.txt
