"""CPU: validate the C oracle's NLMS canceller (no
reference implementation -> "parity unpinned") against an independent
float64 numpy restatement, and check that it actually adapts."""
import numpy as np
import pytest

import oracle as O
from closed_loop import simulate
from conftest import decaying_filters, rel_err, scaled_filters
from nlms_f64 import NlmsF64


@pytest.mark.parametrize("Q,L,N", [(1, 3, 32), (2, 4, 16), (4, 2, 64)])
def test_c_oracle_matches_float64_restatement(Q, L, N):
    rng = np.random.default_rng(Q * 100 + L)
    s = scaled_filters(rng, Q * L, 5 * N + 3, 0.5)
    fc = scaled_filters(rng, Q * L, 3 * N + 2, 0.1)
    kw = dict(gain=0.9, mu=0.05, lam=0.8, delta=1e-3)
    c = O.OracleAuralizer(s, fc, N, Q, L, **kw)
    d = NlmsF64(s, fc, N, Q, L, **kw)
    for b in range(60):
        m = rng.standard_normal((Q, N)).astype(np.float32)
        yc, yd = c.process(m), d.process(m)
        assert rel_err(yc, yd) < 1e-4, b
        assert rel_err(c.feedback_estimate(), d.feedback_estimate()) < 1e-4, b
    W = c.coeffs()
    assert rel_err(W, d.W) < 1e-4
    assert rel_err(c.power(), d.power) < 1e-4


def test_mu_zero_keeps_coefficients():
    rng = np.random.default_rng(2)
    N, L = 32, 2
    s = scaled_filters(rng, L, 100)
    fc = scaled_filters(rng, L, 70, 0.1)
    c = O.OracleAuralizer(s, fc, N, 1, L, mu=0.0)
    W0 = c.coeffs().copy()
    for _ in range(10):
        c.process(rng.standard_normal((1, N)).astype(np.float32))
    assert np.array_equal(W0, c.coeffs())


def erle_run(aur, synth_L, F, N, blocks, seed=1):
    """Closed loop (oracle.hpp:58-122 convention); returns per-block
    feedback energy and residual-feedback energy (feedback - estimate)."""
    L = F.shape[0]
    src = np.random.default_rng(seed).standard_normal((1, blocks * N))
    timeline = np.zeros((1, (blocks + 1) * N + F.shape[1]))
    fb, rr = [], []
    for n in range(blocks):
        f = timeline[:, n * N:(n + 1) * N].copy()
        mic = (src[:, n * N:(n + 1) * N] + f).astype(np.float32)
        est = aur.feedback_estimate()
        fb.append(np.sum(f ** 2))
        rr.append(np.sum((f - est) ** 2))
        spk = aur.process(mic)
        for l in range(L):
            r = np.convolve(spk[l].astype(np.float64), F[l])
            timeline[0, (n + 1) * N:(n + 1) * N + r.size] += r
    return np.array(fb), np.array(rr)


def test_nlms_adapts_closed_loop():
    """F^_0 = 0 in a closed loop with true paths F (loop gain < 1): the
    adaptive canceller must suppress the feedback it starts blind to
    (ERLE over the last 500 blocks > 6 dB; mu = 0 gives exactly 0 dB)."""
    rng = np.random.default_rng(4)
    N, L, blocks = 32, 2, 1500
    synth = decaying_filters(rng, L, 8 * N, scale=0.5)
    F = decaying_filters(rng, L, 2 * N, t60_s=0.002, scale=0.3).astype(np.float64)
    zero = np.zeros((L, 2 * N), np.float32)
    aur = O.OracleAuralizer(synth, zero, N, 1, L, mu=0.002, lam=0.9, delta=1.0)
    fb, rr = erle_run(aur, synth, F, N, blocks)
    erle = 10 * np.log10(fb[-500:].sum() / rr[-500:].sum())
    assert erle > 6.0, erle
    fixed = O.OracleAuralizer(synth, zero, N, 1, L, mu=0.0)
    fb0, rr0 = erle_run(fixed, synth, F, N, 200)
    assert np.allclose(fb0, rr0)


@pytest.mark.parametrize("Q,L,N", [(1, 3, 32), (2, 2, 16)])
def test_constrained_c_oracle_matches_float64_restatement(Q, L, N):
    """Appendix A step 2's constrained variant (c2r -> zero the last N
    samples -> r2c of each gradient) in the C oracle vs numpy float64."""
    rng = np.random.default_rng(Q * 10 + L + 7)
    s = scaled_filters(rng, Q * L, 5 * N + 3, 0.5)
    fc = scaled_filters(rng, Q * L, 3 * N + 2, 0.1)
    kw = dict(gain=0.9, mu=0.05, lam=0.8, delta=1e-3, constrained=True)
    c = O.OracleAuralizer(s, fc, N, Q, L, **kw)
    d = NlmsF64(s, fc, N, Q, L, **kw)
    for b in range(60):
        m = rng.standard_normal((Q, N)).astype(np.float32)
        assert rel_err(c.process(m), d.process(m)) < 1e-4, b
        assert rel_err(c.feedback_estimate(), d.feedback_estimate()) < 1e-4, b
    assert rel_err(c.coeffs(), d.W) < 1e-4


def test_constrained_update_keeps_partitions_causal():
    """The point of the constraint: every W partition stays the spectrum of
    N taps followed by N zeros (as make_partitioned_filters builds it), so
    the canceller stays a linear convolution; the unconstrained gradient
    fills the second half with circular-correlation terms."""
    rng = np.random.default_rng(12)
    N, L = 32, 2
    s = scaled_filters(rng, L, 6 * N, 0.5)
    fc = scaled_filters(rng, L, 3 * N, 0.1)
    tails = {}
    for cons in (False, True):
        c = O.OracleAuralizer(s, fc, N, 1, L, mu=0.05, lam=0.8, delta=1e-3, constrained=cons)
        for _ in range(80):
            c.process(rng.standard_normal((1, N)).astype(np.float32))
        w = np.fft.irfft(c.coeffs().astype(np.complex128), n=2 * N, axis=-1)
        tails[cons] = np.sqrt(np.sum(w[..., N:] ** 2) / np.sum(w[..., :N] ** 2))
    assert tails[True] < 1e-5, tails
    assert tails[False] > 1e-2, tails


def test_constrained_nlms_adapts_closed_loop():
    """The constrained canceller also suppresses closed-loop feedback it
    starts blind to (same setup as test_nlms_adapts_closed_loop)."""
    rng = np.random.default_rng(4)
    N, L, blocks = 32, 2, 1500
    synth = decaying_filters(rng, L, 8 * N, scale=0.5)
    F = decaying_filters(rng, L, 2 * N, t60_s=0.002, scale=0.3).astype(np.float64)
    zero = np.zeros((L, 2 * N), np.float32)
    aur = O.OracleAuralizer(synth, zero, N, 1, L, mu=0.002, lam=0.9, delta=1.0, constrained=True)
    fb, rr = erle_run(aur, synth, F, N, blocks)
    erle = 10 * np.log10(fb[-500:].sum() / rr[-500:].sum())
    assert erle > 6.0, erle
