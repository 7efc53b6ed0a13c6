"""GPU parity at BASELINE.json's full sizes through a size-independent
property: an impulse on one input makes every output the filter itself, so
after K + 1 blocks each loudspeaker's stream must equal its (zero-padded)
synthesis filter -- every partition of every tile, the ring wrap of the
delay line and the tiled spectra layout are exercised at full length.

- c4 shape, MIMO Q = 4 inputs x 16 loudspeakers, 12 s (576k taps), over the
  block-size sweep N = 32 ... 1024 (BASELINE configs[3]);
- c5 shape, 512 loudspeakers, 96 kHz, N = 128, 20 s (1.92M taps, 7.9 GB of
  spectra on the device; 16 distinct filters, aliased).
Tolerance: max |y - h| <= 1e-5 x rms(h) (north star)."""
import numpy as np
import pytest

import paper_2509_04390_b200 as A
from conftest import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-5


def decaying(rng, rows, n, fs):
    env = (10.0 ** (-3.0 * np.arange(n, dtype=np.float64) / n)).astype(np.float32)
    out = np.empty((rows, n), np.float32)
    for r in range(rows):
        h = rng.standard_normal(n, dtype=np.float32) * env
        out[r] = h / np.float32(np.sqrt(np.dot(h.astype(np.float64), h)))
    return out


def impulse_stream(conv, h_of, Q, q_hot, N, blocks, L):
    """Feed an impulse on input q_hot at t = 0; return max |y - h| and rms(h)."""
    worst, ss, cnt = 0.0, 0.0, 0
    x0 = np.zeros((Q, N), np.float32)
    x0[q_hot, 0] = 1.0
    zero = np.zeros((Q, N), np.float32)
    for b in range(blocks):
        y = conv.process(x0 if b == 0 else zero).astype(np.float64)
        ref = h_of(b)  # (L, N) filter samples [bN, (b+1)N), zero-padded
        worst = max(worst, float(np.max(np.abs(y - ref))))
        ss += float(np.sum(ref * ref))
        cnt += ref.size
    return worst, np.sqrt(ss / cnt)


@pytest.mark.parametrize("N", [32, 64, 128, 256, 512, 1024])
def test_c4_mimo_sweep_impulse_full_length(N):
    Q, L, n_h = 4, 16, 576000
    rng = np.random.default_rng(N)
    f = decaying(rng, Q * L, n_h, 48000)  # row q*L + l
    cfg = A.make_config(48000, N, Q, L, mimo=True)
    conv = A.Convolver(list(f), cfg, A.ChannelMode.mimo)
    K = conv.partition_count()
    assert K == -(-n_h // N)
    q_hot = 2
    hq = np.zeros((L, (K + 1) * N), np.float64)
    hq[:, :n_h] = f[q_hot * L:(q_hot + 1) * L]
    worst, rms = impulse_stream(conv, lambda b: hq[:, b * N:(b + 1) * N], Q, q_hot, N, K + 1, L)
    assert worst / rms <= TOL, (worst, rms)


def test_c5_impulse_full_length_512_channels():
    N, L, n_h, fs = 128, 512, 1920000, 96000
    rng = np.random.default_rng(5)
    base = decaying(rng, 16, n_h, fs)
    rows = [base[l % 16] for l in range(L)]
    conv = A.Convolver(rows, A.make_config(fs, N, 1, L), A.ChannelMode.broadcast)
    K = conv.partition_count()
    assert K == 15000
    pad = np.zeros((16, (K + 1) * N), np.float64)
    pad[:, :n_h] = base
    idx = np.arange(L) % 16
    worst, rms = impulse_stream(conv, lambda b: pad[idx, b * N:(b + 1) * N], 1, 0, N, K + 1, L)
    assert worst / rms <= TOL, (worst, rms)
