"""Experiment (GPU box): where the back-to-back block cycle goes at c3 --
per-block CUDA events vs one event pair around all blocks, graph vs stream
launches, and the in-kernel %globaltimer cycle."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2509_04390_b200 as A  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
synth, fc, mic = bench.make_workload(cfg)
e = bench.make_engine(A, cfg, synth, fc, 0)
e.time_device_blocks(50, mic)
res = {}
for mode in (0, 1):
    e.set_launch_mode(mode)
    _, us = e.time_device_blocks(500, mic)
    span = e.time_device_span(500, mic)
    res[f"mode{mode}"] = {"per_block_events_p50": float(np.median(us)), "per_block_events_mean": float(np.mean(us)),
                          "span_mean": span}
e.set_launch_mode(0)
tr = e.trace_blocks(32)
res["trace_cycle_p50"] = float(np.median(tr["cycle"][:, 0])) if "cycle" in tr else None
res["trace"] = {k: [float(np.median(v[:, 0])), float(np.median(v[:, 1]))] for k, v in tr.items()}
print(json.dumps(res))

# the same blocks through process()'s mapped-memory handshake
trh = e.trace_blocks(32, host_inputs=mic)
res2 = {"host_trace_cycle_p50": float(np.median(trh["cycle"][:, 0])) if "cycle" in trh else None,
        "host_trace": {k: [float(np.median(v[:, 0])), float(np.median(v[:, 1]))] for k, v in trh.items()}}
print(json.dumps(res2))
