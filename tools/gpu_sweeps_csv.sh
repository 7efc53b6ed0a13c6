#!/bin/bash
# GPU call: the paper's Section VI sweeps as extended reference CSV.
TAG=${1:-csv}
O=gpurun_out/$TAG
mkdir -p $O
S="timeout -s KILL 600 python tools/sweep_csv.py --trials 1000"
$S --subject convolver --parameter block_size -o $O/convolver_block_size.csv 2> $O/e1.log
$S --subject auralizer --parameter block_size -o $O/auralizer_block_size.csv 2> $O/e2.log
$S --subject auralizer --parameter channels --values 1,2,4,8,16,32,64,128,256,512,1024 -o $O/auralizer_channels.csv 2> $O/e3.log
$S --subject convolver --parameter filter_length_s -o $O/convolver_filter_length.csv 2> $O/e4.log
$S --subject auralizer --parameter fc_length_s -o $O/auralizer_fc_length.csv 2> $O/e5.log
tail -n 3 $O/*.log
