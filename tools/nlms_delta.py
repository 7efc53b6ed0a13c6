"""Measurement (GPU box): canceller coefficient error at the SURVEY
Appendix-A regulariser delta = 1e-6 N versus the engine default 1e-2 * 2N.

For each delta, the same seeded closed-form input stream goes through
  - the GPU engine (C-ABI),
  - the C oracle in fp32 (the parity checker),
  - the independent float64 restatement (tests/nlms_f64.py),
and the W error max|W - W64| / rms(W64) is printed per checkpoint block for
both fp32 implementations: the GPU's error against f64 should be no worse
than ~1.5x the oracle's own (fp32 rounding, not a GPU defect).
    python tools/nlms_delta.py > profiles/r2_nlms_delta.txt
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import paper_2509_04390_b200 as A  # noqa: E402
from conftest import decaying_filters, rel_err  # noqa: E402
from nlms_f64 import NlmsF64  # noqa: E402


def run(N, L, n_h, n_hf, delta, blocks, checkpoints, mu=0.005, lam=0.9, seed=11):
    rng = np.random.default_rng(seed)
    synth = decaying_filters(rng, L, n_h)
    fc = decaying_filters(rng, L, n_hf, t60_s=0.3, scale=0.1)
    g = A.Auralizer(list(synth), list(fc), A.make_config(48000, N, 1, L),
                    afc=A.AfcParams(mu, lam, delta))
    o = O.OracleAuralizer(synth, fc, N, 1, L, mu=mu, lam=lam, delta=delta)
    d = NlmsF64(synth, fc, N, 1, L, mu=mu, lam=lam, delta=delta)
    rows = []
    for b in range(1, blocks + 1):
        m = rng.standard_normal((1, N)).astype(np.float32)
        yg, yo, yd = g.process(m), o.process(m), d.process(m)
        if b in checkpoints:
            Wd = d.W[0]
            Wg, Wo = g.coeffs()[0], o.coeffs()[0]
            rows.append(dict(block=b, delta=delta, N=N, L=L,
                             W_gpu_vs_f64=rel_err(Wg, Wd), W_oracle_vs_f64=rel_err(Wo, Wd),
                             W_gpu_vs_oracle=rel_err(Wg, Wo),
                             y_gpu_vs_f64=rel_err(yg, yd), y_oracle_vs_f64=rel_err(yo, yd),
                             y_gpu_vs_oracle=rel_err(yg, yo)))
            l, k, j = np.unravel_index(int(np.argmax(np.abs(Wg - Wo))), Wg.shape)
            pw = o.power()
            rows[-1].update(worst_lkj=[int(l), int(k), int(j)], power_at_worst=float(pw[j]),
                            power_min=float(pw.min()), power_median=float(np.median(pw)))
            print(json.dumps(rows[-1]), flush=True)
    g.close()
    return rows


if __name__ == "__main__":
    cps = {1, 2, 5, 10, 20, 50, 100, 200}
    if sys.argv[1:] == ["c3"]:  # BASELINE configs[2] at full size (10 s synthesis)
        for delta in (1e-6 * 64, 1e-2 * 2 * 64, 1.0):
            run(64, 64, 480000, 48000, delta, 200, {1, 2, 10, 50, 100, 200}, seed=2024)
        sys.exit(0)
    for (N, L, n_h, n_hf) in [(64, 8, 64 * 40, 64 * 40), (64, 64, 64 * 40, 48000)]:
        for delta in (1e-6 * N, 1e-2 * 2 * N):
            run(N, L, n_h, n_hf, delta, 200, cps)
