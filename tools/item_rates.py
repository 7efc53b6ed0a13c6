#!/usr/bin/env python
"""Per-item streaming rates of k_back from its per-item trace (c3 shape):
bytes each item streams / (partial written - item start), by kind and phase."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_04390_b200 as A  # noqa: E402


def main():
    N, L = 64, 64
    rng = np.random.default_rng(0)
    base = rng.standard_normal((16, 480000), dtype=np.float32) * np.float32(1e-3)
    basef = rng.standard_normal((16, 48000), dtype=np.float32) * np.float32(1e-4)
    e = A.Auralizer([base[i % 16] for i in range(L)], [basef[i % 16] for i in range(L)],
                    A.make_config(48000, N, 1, L), afc=A.AfcParams(0.005, 0.9, None))
    mic = rng.standard_normal((64, 1, N)).astype(np.float32)
    e.time_device_blocks(50, mic)
    segs, ctas = e.trace_back(8)
    NF, CT, LT = N // 2, 32, 8
    # bytes per item: synthesis tap rows (LT + 1) x CT float4; canceller units
    # (2P W + ~1 XA row) x CT float4 (P = 1)
    kind, b, en, cta, t0, tp, t1 = segs[:, 0], segs[:, 2], segs[:, 3], segs[:, 4], segs[:, 5], segs[:, 6], segs[:, 7]
    items = en - b
    byts = np.where(kind == 0, items * (LT + 1) * CT * 16, items * 3 * CT * 16)
    dur = tp - t0
    out = {}
    for k, nm in ((0, "synthesis"), (1, "canceller")):
        m = (kind == k) & (dur > 0)
        r = byts[m] / (dur[m] * 1e-6) / 1e9
        out[nm] = {"items": int(m.sum()), "MB": float(byts[m].sum() / 1e6),
                   "GBps_per_SM_p10_50_90": [round(float(np.percentile(r, x)), 1) for x in (10, 50, 90)],
                   "start_us_p10_50_90": [round(float(np.percentile(t0[m], x)), 1) for x in (10, 50, 90)]}
    # aggregate throughput over time: bytes of items completed per 5 us window
    order = np.argsort(tp)
    hist = np.histogram(tp, bins=np.arange(0, 65, 5), weights=byts)[0] / 5e-6 / 1e9
    out["aggregate_GBps_per_5us_window"] = [round(float(x)) for x in hist]
    out["cta_start_exit_p0_50_100"] = [[round(float(np.percentile(ctas[:, i], x)), 1) for x in (0, 50, 100)]
                                       for i in (0, 2)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
