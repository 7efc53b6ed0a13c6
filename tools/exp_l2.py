"""Experiment (GPU box): k_back on an L2-resident configuration (c2 by
default): launch time, per-CTA start / first data / exit, per-item streaming
rates, and the stage-size knob, to see what keeps it below the L2 read
roofline (profiles/r2_l2_probe.jsonl)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2509_04390_b200 as A  # noqa: E402


def run(cfg_name, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = str(v)
    cfg = dict(bench.CONFIGS[cfg_name])
    Q, L = cfg["Q"], cfg["L"]
    synth = bench.aliased_rows(Q * L, cfg["n_h"])
    fc = bench.aliased_rows(Q * L, cfg["n_hf"], scale=1e-4) if cfg["afc"] else None
    e = bench.make_engine(A, cfg, synth, fc, 0)
    mic = np.random.default_rng(7).standard_normal((64, Q, cfg["N"])).astype(np.float32)
    e.time_device_blocks(50, mic)
    ph = e.profile_phases(5)
    byts = ph["k_back"][1]
    us = e.time_phase("k_back", 50)
    span = e.time_device_span(300, mic)
    segs, ctas = e.trace_back(8)
    dur = segs[:, 6] - segs[:, 5]
    out = {"config": cfg_name, "env": env or {}, "describe": e.describe(), "k_back_bytes": byts,
           "k_back_us": us, "GBps": byts / (us * 1e-6) / 1e9, "block_span_us": span,
           "cta_start_p0_50_100": [float(np.percentile(ctas[:, 0], x)) for x in (0, 50, 100)],
           "cta_first_data_p0_50_100": [float(np.percentile(ctas[:, 1], x)) for x in (0, 50, 100)],
           "cta_exit_p0_50_100": [float(np.percentile(ctas[:, 2], x)) for x in (0, 50, 100)],
           "items": int(segs.shape[0]), "item_us_p10_50_90": [float(np.percentile(dur, x)) for x in (10, 50, 90)]}
    e.close()
    for k in (env or {}):
        os.environ.pop(k)
    return out


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    print(json.dumps(run(name)), flush=True)
    for env in ({"AURA_B200_STAGE_KB": 24}, {"AURA_B200_STAGE_KB": 32}, {"AURA_B200_STAGE_KB": 64},
                {"AURA_B200_QITEMS": 4}, {"AURA_B200_QITEMS": 24}, {"AURA_B200_PHASE_B": 0.95}):
        print(json.dumps(run(name, env)), flush=True)
