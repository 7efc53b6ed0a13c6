#!/usr/bin/env python
"""Host-visible latency of process() (C-ABI, host buffers) in graph mode (0)
and stream-launch mode (1): back to back, and paced on the real-time grid
(one block every N/fs). c3 shape unless --L/--N."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_04390_b200 as A  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--blocks", type=int, default=2000)
    args = ap.parse_args()
    N, L = args.N, args.L
    rng = np.random.default_rng(0)
    base = rng.standard_normal((16, 480000), dtype=np.float32) * np.float32(1e-3)
    basef = rng.standard_normal((16, 48000), dtype=np.float32) * np.float32(1e-4)
    e = A.Auralizer([base[i % 16] for i in range(L)], [basef[i % 16] for i in range(L)],
                    A.make_config(48000, N, 1, L), afc=A.AfcParams(0.005, 0.9, None))
    mic = rng.standard_normal((64, 1, N)).astype(np.float32)
    pace = 1e6 * N / 48000
    q = lambda v: {p: round(float(np.percentile(v, p)), 2) for p in (50, 90, 99)}
    e.set_launch_mode(0)
    for p in (0.0, pace):
        br = e.time_host_breakdown(mic, 1000, pace_us=p)
        print(json.dumps({"breakdown_pace_us": p, "p50": {k: round(float(np.median(v)), 2) for k, v in br.items()},
                          "p99": {k: round(float(np.percentile(v, 99)), 2) for k, v in br.items()}}), flush=True)
    for mode in (0, 1):
        e.set_launch_mode(mode)
        e.time_host_blocks(mic, 200)
        b2b = e.time_host_blocks(mic, args.blocks)
        res = {"mode": mode, "back_to_back_us": q(b2b)}
        for p in (100.0, 200.0, 500.0, pace):
            res[f"paced_{p:.0f}us"] = q(e.time_host_blocks(mic, min(args.blocks, 1000), pace_us=p))
        print(json.dumps(res), flush=True)
    e.close()


if __name__ == "__main__":
    main()
