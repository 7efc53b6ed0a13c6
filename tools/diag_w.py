"""Diagnostic: growth of the canceller-coefficient mismatch (GPU vs C oracle)
at the c3 shape for several regularisers."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
import paper_2509_04390_b200 as A
from conftest import decaying_filters, rel_err

N, L = 64, 64
rng = np.random.default_rng(2024)
synth = decaying_filters(rng, L, 480000)
fc = decaying_filters(rng, L, 48000, t60_s=0.3, scale=0.1)
for delta in (1e-6 * N, 1.0, 100.0):
    kw = dict(mu=0.005, lam=0.9, delta=delta)
    g = A.Auralizer(list(synth), list(fc), A.make_config(48000, N, 1, L),
                    afc=A.AfcParams(0.005, 0.9, delta))
    o = O.OracleAuralizer(synth, fc, N, 1, L, **kw)
    W0 = o.coeffs().copy()
    r = np.random.default_rng(5)
    for b in range(1, 201):
        m = r.standard_normal((1, N)).astype(np.float32)
        y, yo = g.process(m), o.process(m)
        if b in (1, 2, 5, 10, 20, 40, 100, 200):
            Wg, Wo = g.coeffs(), o.coeffs()
            print(f"delta={delta:g} block {b}: out {rel_err(y, yo):.2e} fhat "
                  f"{rel_err(g.feedback_estimate(), o.feedback_estimate()):.2e} W {rel_err(Wg, Wo):.2e} "
                  f"|W-W0|/|W0| {np.linalg.norm(Wo - W0) / np.linalg.norm(W0):.2e}", flush=True)
