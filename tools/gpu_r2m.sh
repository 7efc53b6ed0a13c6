#!/bin/bash
bash tools/gpu_sweep.sh r2sweep
bash tools/gpu_sweeps_csv.sh r2csv
