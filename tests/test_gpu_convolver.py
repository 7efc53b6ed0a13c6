"""GPU parity: the B200 Convolver (through the C-ABI) against the reference
(golden fixtures made by the unmodified reference), the C oracle and the
fp64 direct convolution. Mirrors test_convolver.cpp / verify.hpp.

Tolerance (north star): max|y - y_ref| / rms(y_ref) <= 1e-5 in fp32."""
import numpy as np
import pytest

import oracle as O
import paper_2509_04390_b200 as A
from conftest import decaying_filters, golden, rel_err, scaled_filters

pytestmark = pytest.mark.gpu
TOL = 1e-5


def gpu_conv(filters, N, inputs, outputs, mode):
    mimo = mode == A.ChannelMode.mimo
    cfg = A.make_config(48000, N, inputs, outputs, mimo=mimo)
    return A.Convolver(list(filters), cfg, mode)


@pytest.mark.parametrize("name", ["conv_bcast_n64", "conv_bcast_n128", "conv_elem_n16",
                                  "conv_bcast_n16_h1", "conv_bcast_n256_long"])
def test_golden_reference_outputs(name):
    g = golden(name)
    N, L, mode = int(g["N"]), int(g["L"]), int(g["mode"])
    inputs = 1 if mode == 0 else L
    conv = gpu_conv(g["filters"], N, inputs, L, mode)
    assert conv.partition_count() == int(g["partitions"])
    y = np.stack([conv.process(x) for x in g["x"]])
    assert rel_err(y, g["y"]) <= TOL
    k_show = min(conv.partition_count(), 3)
    spec = np.stack([conv.spectrum(c, k) for c in range(L) for k in range(k_show)])
    # the device r2c performs the reference's float operations: bit-identical
    assert np.array_equal(spec, g["spectra"])
    assert np.all(spec[:, 0].imag == 0) and np.all(spec[:, -1].imag == 0)


GRID = [(N, n_h, C, mode)
        for N in (16, 64, 128)
        for n_h in (1, N - 1, N, N + 1, 3 * N + 7, 10 * N)
        for C in (1, 4)
        for mode in (0, 1)]


@pytest.mark.parametrize("N,n_h,C,mode", GRID)
def test_verify_grid_vs_oracle_and_direct(N, n_h, C, mode):
    """verify.hpp:110-145 grid: streamed K+3 blocks vs the 64-bit direct
    convolution (< 1e-4 abs, the reference's own bar) and vs the C oracle
    (<= 1e-5 rel)."""
    rng = np.random.default_rng(N * 7919 + n_h * 31 + C * 3 + mode)
    f = scaled_filters(rng, C, n_h)
    inputs = 1 if mode == 0 else C
    conv = gpu_conv(f, N, inputs, C, mode)
    orc = O.OracleConvolver(f, N, inputs, C, mode)
    blocks = -(-n_h // N) + 3
    x = rng.standard_normal((blocks, inputs, N)).astype(np.float32)
    y = np.stack([conv.process(b) for b in x])
    yo = np.stack([orc.process(b) for b in x])
    assert rel_err(y, yo) <= TOL
    for c in range(C):
        xin = x[:, 0 if mode == 0 else c].reshape(-1)
        ref = O.direct_convolve(xin, f[c])[:blocks * N]
        assert np.max(np.abs(y[:, c].reshape(-1) - ref)) < 1e-4


def test_impulse_identity_and_one_block_delay():
    # test_convolver.cpp:30-61
    N = 64
    conv = gpu_conv([np.array([1.0], np.float32)], N, 1, 1, 0)
    rng = np.random.default_rng(100)
    for _ in range(5):
        x = rng.standard_normal((1, N)).astype(np.float32)
        assert np.max(np.abs(conv.process(x) - x)) <= 2e-6
    d = np.zeros(N + 1, np.float32)
    d[N] = 1.0
    conv = gpu_conv([d], N, 1, 1, 0)
    prev = np.zeros((1, N), np.float32)
    for _ in range(4):
        x = rng.standard_normal((1, N)).astype(np.float32)
        assert np.max(np.abs(conv.process(x) - prev)) <= 2e-6
        prev = x


def test_unit_partition_spectrum_flat():
    conv = gpu_conv([np.array([1.0], np.float32)], 64, 1, 1, 0)
    s = conv.spectrum(0, 0)
    assert np.max(np.abs(s - 1.0)) <= 1e-6


def test_reset_is_bit_exact_and_idempotent():
    # test_convolver.cpp:172-193
    N = 64
    rng = np.random.default_rng(9)
    conv = gpu_conv(scaled_filters(rng, 1, 200, 0.1 * np.sqrt(200)), N, 1, 1, 0)
    x = rng.standard_normal((1, N)).astype(np.float32)
    fresh = conv.process(x).copy()
    for _ in range(5):
        conv.process(rng.standard_normal((1, N)).astype(np.float32))
    assert conv.blocks_processed() == 6
    conv.reset()
    assert conv.blocks_processed() == 0
    assert np.array_equal(conv.process(x), fresh)
    conv.reset()
    conv.reset()
    assert np.array_equal(conv.process(np.zeros((1, N), np.float32)), np.zeros((1, N)))


def test_first_block_uses_only_partition_zero():
    # test_convolver.cpp:246-269 (bit-exact)
    N = 64
    rng = np.random.default_rng(600)
    head = rng.standard_normal(N).astype(np.float32) * 0.5
    f1 = np.concatenate([head, rng.standard_normal(2 * N).astype(np.float32)])
    f2 = np.concatenate([head, rng.standard_normal(2 * N).astype(np.float32)])
    x = rng.standard_normal((1, N)).astype(np.float32)
    y1 = gpu_conv([f1], N, 1, 1, 0).process(x)
    y2 = gpu_conv([f2], N, 1, 1, 0).process(x)
    assert np.array_equal(y1, y2)


def test_deterministic_across_instances():
    N, L = 64, 16
    rng = np.random.default_rng(5)
    f = scaled_filters(rng, L, 40 * N)
    a, b = gpu_conv(f, N, 1, L, 0), gpu_conv(f, N, 1, L, 0)
    for _ in range(50):
        x = rng.standard_normal((1, N)).astype(np.float32)
        assert np.array_equal(a.process(x), b.process(x))


def test_broadcast_equals_elementwise():
    # test_convolver.cpp:224-244
    N, C = 64, 4
    rng = np.random.default_rng(400)
    f = scaled_filters(rng, C, 3 * N + 7)
    b = gpu_conv(f, N, 1, C, 0)
    e = gpu_conv(f, N, C, C, 1)
    for _ in range(6):
        x = rng.standard_normal((1, N)).astype(np.float32)
        yb = b.process(x)
        ye = e.process(np.repeat(x, C, axis=0))
        assert np.max(np.abs(yb - ye)) <= 1e-6


def test_linearity():
    N, n_h = 64, 150
    rng = np.random.default_rng(7)
    f = scaled_filters(rng, 1, n_h)
    cx, cy, cm = (gpu_conv(f, N, 1, 1, 0) for _ in range(3))
    for _ in range(3):
        x = rng.standard_normal((1, N)).astype(np.float32)
        y = rng.standard_normal((1, N)).astype(np.float32)
        om = cm.process((0.8 * x - 1.3 * y).astype(np.float32))
        assert np.max(np.abs(om - (0.8 * cx.process(x) - 1.3 * cy.process(y)))) <= 1e-4


@pytest.mark.parametrize("Q,L,N,n_h", [(4, 8, 64, 20 * 64 + 3), (2, 3, 32, 100), (4, 64, 32, 2000)])
def test_mimo_vs_oracle(Q, L, N, n_h):
    rng = np.random.default_rng(Q * L)
    f = decaying_filters(rng, Q * L, n_h)
    conv = gpu_conv(f, N, Q, L, A.ChannelMode.mimo)
    orc = O.OracleConvolver(f, N, Q, L, O.MIMO)
    blocks = -(-n_h // N) + 3
    x = rng.standard_normal((blocks, Q, N)).astype(np.float32)
    y = np.stack([conv.process(b) for b in x])
    yo = np.stack([orc.process(b) for b in x])
    assert rel_err(y, yo) <= TOL


def test_error_codes():
    cfg = A.make_config(48000, 64, 1, 1)
    conv = A.Convolver([np.ones(3, np.float32)], cfg)
    with pytest.raises(A.Error) as ei:
        conv.process(np.zeros((2, 64), np.float32))
    assert ei.value.code == A.ErrorCode.shape_mismatch
    with pytest.raises(A.Error) as ei:
        conv.process(np.zeros((1, 32), np.float32))
    assert ei.value.code == A.ErrorCode.shape_mismatch
    bad = np.zeros((1, 64), np.float32)
    bad[0, 7] = np.inf
    with pytest.raises(A.Error) as ei:
        conv.process(bad)
    assert ei.value.code == A.ErrorCode.non_finite_input
    assert conv.blocks_processed() == 0
    with pytest.raises(A.Error) as ei:
        A.Convolver([np.ones(3)] * 2, A.make_config(48000, 64, 2, 2), A.ChannelMode.broadcast)
    assert ei.value.code == A.ErrorCode.mode_channel_mismatch
    with pytest.raises(A.Error) as ei:
        A.Convolver([np.ones(3)], A.make_config(48000, 64, 1, 2))
    assert ei.value.code == A.ErrorCode.mode_channel_mismatch


def test_backend_listing_on_gpu():
    b = A.list_backends()
    assert len(b) >= 1 and b[0].kind == A.BackendKind.accelerator and "B200" in b[0].detail
    assert A.make_backend("gpu").device == 0


def test_c2_full_size_channel_subset_vs_oracle():
    """configs[1]: 1 x 16 loudspeakers, N = 128, 10 s (480k taps), K = 3750,
    streamed K + 3 blocks on the GPU; channels {0, 15} re-run on the C oracle
    (synthesis channels are independent)."""
    N, L, n_h = 128, 16, 480000
    rng = np.random.default_rng(1000)
    f = decaying_filters(rng, L, n_h)
    conv = gpu_conv(f, N, 1, L, 0)
    assert conv.partition_count() == 3750
    sub = [0, L - 1]
    orc = O.OracleConvolver(f[sub], N, 1, len(sub), O.BROADCAST)
    blocks = 3750 + 3
    worst = 0.0
    ys, yos = [], []
    for b in range(blocks):
        x = rng.standard_normal((1, N)).astype(np.float32)
        y = conv.process(x)
        ys.append(y[sub])
        yos.append(orc.process(x))
    assert rel_err(np.stack(ys), np.stack(yos)) <= TOL
