#!/bin/bash
O=gpurun_out/r2q
mkdir -p $O
timeout 600 python tools/item_rates.py > $O/item_rates.json 2> $O/item_rates.err
cat $O/item_rates.json; tail -3 $O/item_rates.err
