"""Experiment (GPU box): process() latency at c3 on the real-time grid and
back to back, block graph (launch mode 0) vs stream launches (mode 1), two
repetitions: {mode_rep: [paced p50, p99, b2b p50, p99]} in us."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import bench
import paper_2509_04390_b200 as A
cfg = dict(bench.CONFIGS["c3"])
Q, L = cfg["Q"], cfg["L"]
e = bench.make_engine(A, cfg, bench.aliased_rows(Q * L, cfg["n_h"]), bench.aliased_rows(Q * L, cfg["n_hf"], scale=1e-4), 0)
mic = np.random.default_rng(7).standard_normal((64, Q, cfg["N"])).astype(np.float32)
out = {}
for rep in range(2):
    for mode in (0, 1):
        e.set_launch_mode(mode)
        e.time_host_blocks(mic, 100, pace_us=1333.333)
        us = e.time_host_blocks(mic, 1500, pace_us=1333.333)
        b2b = e.time_host_blocks(mic, 500)
        out[f"{mode}_{rep}"] = [round(float(np.percentile(us, q)), 2) for q in (50, 99)] + [round(float(np.percentile(b2b, q)), 2) for q in (50, 99)]
print(json.dumps(out))
