#!/usr/bin/env python
"""Ablation of the streaming kernel k_back on one GPU: device time of the
kernel alone (time_phase) and the in-graph timeline, for the c3 shape with
and without the canceller / NLMS, and a canceller-only engine.

    python tools/exp_back.py [--L 64] [--N 64]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_04390_b200 as A  # noqa: E402


MODE = 0


def run(name, eng, mic, blocks=200):
    eng.set_launch_mode(MODE)
    eng.time_device_blocks(20, mic)
    lat, us = eng.time_device_blocks(blocks, mic)
    tr = eng.trace_blocks(16)
    back = eng.time_phase("k_back", 20)
    byts = eng.profile_phases(5)["k_back"][1]
    segs, ctas = eng.trace_back(8)
    q = lambda v: [round(float(np.percentile(v, x)), 2) for x in (0, 10, 50, 90, 100)]
    kinds = {}
    for kind in (0, 1):
        m = segs[:, 0] == kind
        if m.any():
            nm = "syn" if kind == 0 else "afc"
            kinds[nm + "_end"] = q(segs[m, 7])
            kinds[nm + "_stream_us"] = q(segs[m, 6] - segs[m, 5])
            kinds[nm + "_epilogue_us"] = q(segs[m, 7] - segs[m, 6])
    last = segs[np.argsort(segs[:, 7])[-4:]]
    kinds["last4_items(kind,tile,b,e,cta,start,partial,end)"] = np.round(last, 2).tolist()
    per_cta = np.bincount(segs[:, 4].astype(int), minlength=ctas.shape[0])
    kinds["chunks_per_cta_min_max"] = [int(per_cta.min()), int(per_cta.max())]
    # per CTA: end of its last segment of each phase (A synth, canceller, B synth)
    cta_trace = {"start": q(ctas[:, 0]), "first_data": q(ctas[:, 1]), "exit": q(ctas[:, 2]),
                 "seg_end_by_kind": kinds}
    out = {"case": name, "block_p50_us": float(np.median(us)), "k_back_us": back,
           "k_back_GBps": byts / back / 1e3, "MB": byts / 1e6,
           "timeline": {k: [round(float(np.median(v[:, 0])), 2), round(float(np.median(v[:, 1])), 2)]
                        for k, v in tr.items()},
           "cta_trace_pct_0_10_50_90_100": cta_trace, "engine": eng.describe()}
    print(json.dumps(out), flush=True)
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--cases", default="nlms,cons,mu0,synth,afc")
    ap.add_argument("--mode", type=int, default=0, help="0 graph per block, 1 stream launches")
    args = ap.parse_args()
    global MODE
    MODE = args.mode
    N, L = args.N, args.L
    rng = np.random.default_rng(0)
    n_h, n_hf = 480000, 48000
    base = rng.standard_normal((16, n_h), dtype=np.float32) * np.float32(1e-3)
    basef = rng.standard_normal((16, n_hf), dtype=np.float32) * np.float32(1e-4)
    synth = [base[i % 16] for i in range(L)]
    fc = [basef[i % 16] for i in range(L)]
    mic = rng.standard_normal((64, 1, N)).astype(np.float32)
    cfg = A.make_config(48000, N, 1, L)
    cases = args.cases.split(",")
    if "nlms" in cases:
        run("c3 nlms", A.Auralizer(synth, fc, cfg, afc=A.AfcParams(0.005, 0.9, None)), mic)
    if "cons" in cases:
        run("c3 nlms constrained", A.Auralizer(synth, fc, cfg, afc=A.AfcParams(0.005, 0.9, None, True)), mic)
    if "mu0" in cases:
        run("c3 mu=0", A.Auralizer(synth, fc, cfg, afc=A.AfcParams(0.0, 0.9, None)), mic)
    if "synth" in cases:
        run("synth only", A.Convolver(synth, cfg), mic)
    if "afc" in cases:
        short = [b[:N] for b in synth]
        run("canceller only (K=1)", A.Auralizer(short, fc, cfg, afc=A.AfcParams(0.005, 0.9, None)), mic)


if __name__ == "__main__":
    main()
