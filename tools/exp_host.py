"""Experiment (GPU box): where process()'s host-visible latency goes at c3,
paced on the real-time grid and back to back (time_host_breakdown)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2509_04390_b200 as A  # noqa: E402

cfg = dict(bench.CONFIGS["c3"])
Q, L = cfg["Q"], cfg["L"]
e = bench.make_engine(A, cfg, bench.aliased_rows(Q * L, cfg["n_h"]),
                      bench.aliased_rows(Q * L, cfg["n_hf"], scale=1e-4), 0)
mic = np.random.default_rng(7).standard_normal((64, Q, cfg["N"])).astype(np.float32)
e.time_host_blocks(mic, 200)
out = {}
for pace in (1333.333, 0.0):
    br = e.time_host_breakdown(mic, 1000, pace_us=pace)
    out["paced" if pace else "b2b"] = {k: [round(float(np.percentile(v, q)), 2) for q in (50, 99)] for k, v in br.items()}
tr = e.trace_blocks(32, host_inputs=mic)
out["host_trace_output_us"] = [round(float(np.median(tr["output"][:, 0])), 2), round(float(np.median(tr["output"][:, 1])), 2)]
print(json.dumps(out))
