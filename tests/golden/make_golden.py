"""Regenerate tests/golden/*.npz from the UNMODIFIED reference.

Runs only in a container that has /root/reference (the reference headers are
compiled into oracle/_ref/libaura_ref.so by oracle/Makefile). The fixtures
are small, committed, and used on the GPU box (where /root/reference does not
exist) to pin both the C oracle and the CUDA product.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from conftest import c1_inputs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def filters(rng, rows, n, scale=None):
    s = 1.0 / np.sqrt(n) if scale is None else scale
    return (rng.standard_normal((rows, n)) * s).astype(np.float32)


def conv_case(name, N, n_h, L, mode, blocks, seed):
    rng = np.random.default_rng(seed)
    inputs = 1 if mode == O.BROADCAST else L
    f = filters(rng, L, n_h)
    x = rng.standard_normal((blocks, inputs, N)).astype(np.float32)
    ref = O.RefConvolver(f, N, inputs, L, mode)
    y = np.stack([ref.process(x[b]) for b in range(blocks)])
    spec = np.stack([ref.spectrum(c, k) for c in range(L)
                     for k in range(min(ref.partitions, 3))])
    np.savez_compressed(os.path.join(OUT, name + ".npz"), N=N, n_h=n_h, L=L, mode=mode,
                        filters=f, x=x, y=y, spectra=spec,
                        partitions=ref.partitions)


def aur_case(name, N, n_h, n_hf, L, blocks, gain, seed, fc_scale=1.0):
    rng = np.random.default_rng(seed)
    s = filters(rng, L, n_h)
    fc = filters(rng, L, n_hf) * np.float32(fc_scale)
    m = rng.standard_normal((blocks, 1, N)).astype(np.float32)
    ref = O.RefAuralizer(s, fc, N, L, gain=gain)
    ys, fh = [], []
    for b in range(blocks):
        ys.append(ref.process(m[b]))
        fh.append(ref.feedback_estimate())
    np.savez_compressed(os.path.join(OUT, name + ".npz"), N=N, L=L, gain=gain,
                        synth=s, fc=fc, mic=m, y=np.stack(ys), fhat=np.stack(fh))


def fft_case():
    rng = np.random.default_rng(11)
    d = {}
    for nf in (32, 64, 256, 1024):
        x = rng.standard_normal(nf).astype(np.float32)
        X = O.ref_forward(x)
        d[f"x{nf}"] = x
        d[f"X{nf}"] = X
        d[f"xi{nf}"] = O.ref_inverse(X)
    imp = np.zeros(64, np.float32)
    imp[0] = 1.0
    d["impulse64"] = O.ref_forward(imp)
    np.savez_compressed(os.path.join(OUT, "fft.npz"), **d)


def direct_case():
    y = O.ref_direct_convolve([1, 2, 3], [1, 1])
    rng = np.random.default_rng(5)
    x = rng.standard_normal(100)
    h = rng.standard_normal(37)
    np.savez_compressed(os.path.join(OUT, "direct.npz"), kat=y, x=x, h=h,
                        y=O.ref_direct_convolve(x, h))


def c1_case():
    """BASELINE configs[0] at its exact size: 1 input x 2 loudspeakers, 48 kHz,
    N = 256, 2 s decaying-noise IRs (96,000 taps), K + 3 = 378 blocks of N(0,1)
    input through the reference Convolver. Inputs are regenerated from their
    seeds (tests/conftest.py c1_inputs), so only the output is stored."""
    N, L, n_h, blocks, filt, x = c1_inputs()
    ref = O.RefConvolver(filt, N, 1, L, O.BROADCAST)
    assert ref.partitions == 375
    y = np.stack([ref.process(x[b]) for b in range(blocks)])
    np.savez_compressed(os.path.join(OUT, "c1_full.npz"), N=N, L=L, n_h=n_h, blocks=blocks, y=y)


if __name__ == "__main__":
    if sys.argv[1:] == ["c1"]:
        c1_case()
        sys.exit(0)
    c1_case()
    fft_case()
    direct_case()
    conv_case("conv_bcast_n64", 64, 300, 3, O.BROADCAST, 8, 1)
    conv_case("conv_bcast_n128", 128, 1280, 4, O.BROADCAST, 13, 2)
    conv_case("conv_elem_n16", 16, 55, 4, O.ELEMENTWISE, 7, 3)
    conv_case("conv_bcast_n16_h1", 16, 1, 4, O.BROADCAST, 4, 4)
    conv_case("conv_bcast_n256_long", 256, 96 * 256 + 17, 2, O.BROADCAST, 100, 5)
    aur_case("aur_n64", 64, 5 * 64 + 3, 2 * 64 + 1, 3, 12, 1.0, 6)
    aur_case("aur_n32_gain", 32, 300, 200, 2, 20, 0.7, 7, fc_scale=0.1)
    aur_case("aur_n128_long", 128, 40 * 128, 4 * 128, 8, 50, 1.0, 8, fc_scale=0.1)
    print("golden fixtures written to", OUT)
