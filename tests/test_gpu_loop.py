"""GPU: the persistent block-loop kernel (launch mode 2, loop.cuh) against
the graph mode. The loop runs the same arithmetic in the same order -- the
front's transforms, the streaming work plan and its stage cuts, the
fixed-order split-K reduction -- so outputs, f^ and the canceller spectra
must be BIT-IDENTICAL to the graph mode, block for block, including across
mode switches (the window history flips buffers with the block parity) and
after reset()."""
import numpy as np
import pytest

import paper_2509_04390_b200 as A
from conftest import decaying_filters

pytestmark = pytest.mark.gpu


def make(kind, N, Q, L, n_h, rng, mu=0.01):
    if kind == "aur":
        synth = decaying_filters(rng, Q * L, n_h)
        fc = decaying_filters(rng, Q * L, 4 * N + 3, t60_s=0.01, scale=0.1)
        cfg = A.make_config(48000, N, Q, L, mimo=Q > 1)

        def build():
            return A.Auralizer(list(synth), list(fc), cfg, afc=A.AfcParams(mu, 0.9, None))
    else:
        mode = {"bcast": A.ChannelMode.broadcast, "elem": A.ChannelMode.elementwise,
                "mimo": A.ChannelMode.mimo}[kind]
        f = decaying_filters(rng, (Q * L) if kind == "mimo" else L, n_h)
        cfg = A.make_config(48000, N, Q, L, mimo=kind == "mimo")

        def build():
            return A.Convolver(list(f), cfg, mode)
    return build


def run(eng, xs, modes):
    ys, fs = [], []
    for b, x in enumerate(xs):
        if b in modes:
            eng.set_launch_mode(modes[b])
        ys.append(eng.process(x))
        if isinstance(eng, A.Auralizer):
            fs.append(eng.feedback_estimate())
    return np.stack(ys), (np.stack(fs) if fs else None)


CASES = [("aur", 64, 1, 8, 40 * 64 + 7, 0.01), ("aur", 64, 4, 8, 20 * 64, 0.01),
         ("aur", 256, 1, 4, 9 * 256, 0.0), ("bcast", 128, 1, 12, 30 * 128 + 1, 0.0),
         ("elem", 64, 6, 6, 17 * 64, 0.0), ("mimo", 32, 3, 8, 50 * 32, 0.0)]


@pytest.mark.parametrize("kind,N,Q,L,n_h,mu", CASES)
def test_loop_mode_is_bit_identical_to_graph_mode(kind, N, Q, L, n_h, mu):
    rng = np.random.default_rng(N + Q * 7 + L)
    build = make(kind, N, Q, L, n_h, rng, mu)
    xs = [rng.standard_normal((Q if kind != "elem" else L, N)).astype(np.float32) for _ in range(90)]
    g, lp = build(), build()
    yg, fg = run(g, xs, {})
    # graph for 37 blocks (odd: the loop starts on the second history buffer),
    # loop for 40, graph again, loop again
    yl, fl = run(lp, xs, {37: 2, 77: 0, 83: 2})
    assert np.array_equal(yg, yl)
    if fg is not None:
        assert np.array_equal(fg, fl)
        assert np.array_equal(g.coeffs(), lp.coeffs())
    assert lp.launch_mode() == 2
    g.close()
    lp.close()


def test_loop_mode_reset_replays_exactly():
    rng = np.random.default_rng(5)
    build = make("aur", 64, 1, 8, 30 * 64, rng)
    e = build()
    e.set_launch_mode(2)
    xs = [rng.standard_normal((1, 64)).astype(np.float32) for _ in range(25)]
    first, _ = run(e, xs, {})
    e.reset()
    again, _ = run(e, xs, {})
    assert np.array_equal(first, again)
    e.close()


def test_loop_mode_device_timing_and_c3_shape():
    """c3 shape (1 x 64, N = 64, 10 s, NLMS canceller 1 s): 40 blocks bit-identical
    to the graph mode, then the loop's own device timing runs."""
    N, L = 64, 64
    rng = np.random.default_rng(64)
    synth = decaying_filters(rng, L, 480000)
    fc = decaying_filters(rng, L, 48000, t60_s=0.3, scale=0.1)
    cfg = A.make_config(48000, N, 1, L)
    mk = lambda: A.Auralizer(list(synth), list(fc), cfg, afc=A.AfcParams(0.005, 0.9, None))
    g, lp = mk(), mk()
    lp.set_launch_mode(2)
    xs = [rng.standard_normal((1, N)).astype(np.float32) for _ in range(40)]
    yg, fg = run(g, xs, {})
    yl, fl = run(lp, xs, {})
    assert np.array_equal(yg, yl) and np.array_equal(fg, fl)
    lat, us = lp.time_device_blocks(200, np.stack(xs))
    assert us.shape == (200,) and np.all(us > 0) and np.all(lat > 0) and np.all(lat < us)
    assert float(np.median(us)) < 1333.0  # inside the real-time budget
    g.close()
    lp.close()
