import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running parity run")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def rel_err(y, ref):
    """max |y - ref| / rms(ref): the north-star parity metric."""
    y = np.asarray(y)
    ref = np.asarray(ref)
    if np.iscomplexobj(y) or np.iscomplexobj(ref):
        y, ref = y.astype(np.complex128), ref.astype(np.complex128)
    else:
        y, ref = y.astype(np.float64), ref.astype(np.float64)
    rms = np.sqrt(np.mean(np.abs(ref) ** 2))
    if rms == 0.0:
        return float(np.max(np.abs(y))) if y.size else 0.0
    return float(np.max(np.abs(y - ref)) / rms)


def scaled_filters(rng, rows, n, scale=1.0):
    """verify.hpp:26-36 style: N(0,1)/sqrt(n_h) (times an extra scale)."""
    return (rng.standard_normal((rows, n)) * (scale / np.sqrt(n))).astype(np.float32)


def decaying_filters(rng, rows, n, fs=48000, t60_s=None, scale=1.0):
    """exponentially decaying noise, -60 dB at t60, sum h^2 = 1."""
    t60 = n / fs if t60_s is None else t60_s
    t = np.arange(n) / fs
    env = 10.0 ** (-3.0 * t / t60)
    h = rng.standard_normal((rows, n)) * env
    h /= np.sqrt(np.sum(h * h, axis=1, keepdims=True))
    return (h * scale).astype(np.float32)


def c1_inputs():
    """BASELINE configs[0] inputs (SURVEY 8(d) seeds): 2 decaying-noise IRs of
    96,000 taps (seed 1000) and K + 3 = 378 blocks of N(0,1) input (seed 7)."""
    N, L, n_h = 256, 2, 96000
    blocks = -(-n_h // N) + 3
    filt = decaying_filters(np.random.default_rng(1000), L, n_h)
    x = np.random.default_rng(7).standard_normal((blocks, 1, N)).astype(np.float32)
    return N, L, n_h, blocks, filt, x
