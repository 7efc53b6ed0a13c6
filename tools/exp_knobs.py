"""Experiment (GPU box): block cycle of a configuration under tuning-knob
settings (AURA_B200_* env, read at engine creation): span mean (one event
pair around 300 blocks), %globaltimer cycle and the kernel timeline.
    python tools/exp_knobs.py c3 '{}' '{"AURA_B200_AFC_ROUNDS": 1}' ..."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2509_04390_b200 as A  # noqa: E402


def run(name, env):
    env = dict(env)
    mode = int(env.pop("MODE", 0))  # launch mode (0 graph, 1 stream launches)
    for k, v in env.items():
        os.environ[k] = str(v)
    cfg = dict(bench.CONFIGS[name])
    Q, L = cfg["Q"], cfg["L"]
    synth = bench.aliased_rows(Q * L, cfg["n_h"])
    fc = bench.aliased_rows(Q * L, cfg["n_hf"], scale=1e-4) if cfg["afc"] else None
    e = bench.make_engine(A, cfg, synth, fc, 0)
    e.set_launch_mode(mode)
    mic = np.random.default_rng(7).standard_normal((64, Q, cfg["N"])).astype(np.float32)
    e.time_device_blocks(50, mic)
    spans = [e.time_device_span(300, mic) for _ in range(3)]
    _, us = e.time_device_blocks(300, mic)
    tr = e.trace_blocks(32)
    host = e.time_host_blocks(mic, 300)
    out = {"env": dict(env, MODE=mode), "span_mean_us": float(np.median(spans)), "events_p50": float(np.median(us)),
           "events_p99": float(np.percentile(us, 99)), "e2e_p50": float(np.median(host)),
           "e2e_p99": float(np.percentile(host, 99)),
           "trace": {k: [round(float(np.median(v[:, 0])), 2), round(float(np.median(v[:, 1])), 2)]
                     for k, v in tr.items()}, "describe": e.describe()[-200:]}
    e.close()
    for k in env:
        os.environ.pop(k)
    return out


if __name__ == "__main__":
    name = sys.argv[1]
    for s in sys.argv[2:]:
        print(json.dumps(run(name, json.loads(s))), flush=True)
