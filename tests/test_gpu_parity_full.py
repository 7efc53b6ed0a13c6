"""GPU parity at BASELINE.json's sizes over full-length streams.

SURVEY 8(d)'s parity plan: every partition takes part only after K + 3
blocks, so each configuration streams at least that many blocks (the
reference's own bar: verify.hpp:40-92 streams K + extra_blocks (3) blocks
against its oracle; acceptance_main.cpp:103-138 checks a 10 s filter). The
checkers are the unmodified reference (oracle/_ref, the parallel backend)
wherever it has the feature, else the C oracle (NLMS, MIMO). Inputs are
N(0,1) noise (seed 7 family), synthesis IRs exponentially decaying noise
with T60 = IR length, canceller paths T60 0.3 s x 0.1.

Tolerance. The north star asks max |y - y_ref| <= 1e-5 x rms(y_ref). At
these lengths the fp32 CPU reference is itself ~1e-5 x RMS away from the
exact result -- its sequential accumulation over K ~ 10^4 partitions
(backend.hpp:212-235) drifts (c5: 1.5e-5 against a float64 FFT convolution,
measured) -- so ANY other summation order differs from it by about that
much. Every stream is therefore also run through the float64 build of the
same algorithm (oracle/liboracle64.so, exact twiddles; the ground truth) and
each test asserts, over every streamed sample:
  (1) GPU vs truth       <= max(1e-5, 1.5 x fp32 checker vs truth)
      -- the GPU is as accurate as the reference (up to the 1.5x margin of
         SURVEY App. A's fp32-vs-f64 check), within 1e-5 wherever it is;
  (2) GPU vs fp32 checker <= 1e-5 + (fp32 checker vs truth)
      -- parity with the reference up to the reference's own rounding.
The same two rules apply to the canceller W after the stream.

  c1  1 x 2,   N 256, 96k taps, no canceller       378 blocks (K+3) vs reference + fixture
  c3  1 x 64,  N 64, 480k taps, 48k-tap canceller 7503 blocks (K+3) vs reference (fixed F^)
  c3  same, NLMS mu = 0.005 (survey delta)         753 blocks (K_f+3) vs C oracle, y f^ W
  c4  4 x 64 MIMO, 576k taps, NLMS                 N 64: 753 blocks, N 1024: 566 (K+3) vs C oracle
  c5  1 x 512, 96 kHz, N 128, 1.92M taps          15003 blocks (K+3), every channel, shards 1/2/4/8
"""
import numpy as np
import pytest

import oracle as O
import paper_2509_04390_b200 as A
from conftest import c1_inputs, decaying_filters, golden

pytestmark = pytest.mark.gpu
TOL = 1e-5


class Track:
    """Running max |y - ref| and rms(ref) over a stream (rel_err of the whole
    stream without keeping it)."""

    def __init__(self):
        self.worst, self.ss, self.n = 0.0, 0.0, 0

    def add(self, y, ref):
        y = np.asarray(y, np.float64)
        ref = np.asarray(ref, np.float64)
        self.worst = max(self.worst, float(np.max(np.abs(y - ref))))
        self.ss += float(np.sum(ref * ref))
        self.n += ref.size

    @property
    def rel(self):
        return self.worst / np.sqrt(self.ss / self.n)


class Tri:
    """GPU, fp32 checker and float64 truth over a stream: the three pairwise
    errors, each relative to rms(truth)."""

    def __init__(self):
        self.gx, self.rx, self.gr = Track(), Track(), Track()

    def add(self, gpu, ref, truth):
        truth = np.asarray(truth, np.float64)
        self.gx.add(gpu, truth)
        self.rx.add(ref, truth)
        self.gr.worst = max(self.gr.worst, float(np.max(np.abs(np.asarray(gpu, np.float64) -
                                                                np.asarray(ref, np.float64)))))
        self.gr.ss, self.gr.n = self.gx.ss, self.gx.n

    def report(self):
        return {"gpu_vs_truth": self.gx.rel, "ref_vs_truth": self.rx.rel, "gpu_vs_ref": self.gr.rel}

    def check(self, what, factor=1.5):
        r = self.report()
        print(what, r)
        assert r["gpu_vs_truth"] <= max(TOL, factor * r["ref_vs_truth"]), (what, r)
        assert r["gpu_vs_ref"] <= TOL + r["ref_vs_truth"], (what, r)


def w_tri(Wg, Wr, Wx):
    """Tri of the canceller spectra (relative to rms of the truth's W)."""
    t = Tri()
    t.add(Wg.astype(np.complex128).view(np.float64), Wr.astype(np.complex128).view(np.float64),
          Wx.astype(np.complex128).view(np.float64))
    return t


def noise_blocks(seed, Q, N):
    rng = np.random.default_rng(seed)
    while True:
        yield rng.standard_normal((Q, N)).astype(np.float32)


def c3_filters(L=64, n_h=480000, n_hf=48000, seed=1000):
    rng = np.random.default_rng(seed)
    return (decaying_filters(rng, L, n_h),
            decaying_filters(rng, L, n_hf, t60_s=0.3, scale=0.1))


def test_c1_exact_size_vs_reference():
    """BASELINE configs[0] at its exact size (375 partitions, 378 blocks)
    against the committed reference fixture and the live reference."""
    N, L, n_h, blocks, filt, x = c1_inputs()
    g = golden("c1_full")
    conv = A.Convolver(list(filt), A.make_config(48000, N, 1, L))
    assert conv.partition_count() == 375
    ref = O.RefConvolver(filt, N, 1, L, O.BROADCAST, backend="parallel")
    truth = O.OracleConvolver(filt, N, 1, L, O.BROADCAST, f64=True)
    t_fix, t = Track(), Tri()
    for b in range(blocks):
        y = conv.process(x[b])
        t_fix.add(y, g["y"][b])
        t.add(y, ref.process(x[b]), truth.process(x[b]))
    assert t_fix.rel <= TOL, t_fix.rel
    t.check("c1")
    assert t.report()["gpu_vs_ref"] <= TOL  # K = 375: the plain north-star bar holds


def test_c3_full_stream_vs_reference():
    """configs[2] with the reference's fixed-F^ canceller (mu = 0): all 7503
    blocks (K + 3: the last partitions of every loudspeaker and of the
    canceller's delay line take part) against the unmodified reference
    Auralizer; outputs every block, f^ every 250 blocks."""
    N, L = 64, 64
    synth, fc = c3_filters()
    g = A.Auralizer(list(synth), list(fc), A.make_config(48000, N, 1, L), afc=A.AfcParams(0.0))
    assert g.synth_partitions() == 7500 and g.fc_partitions() == 750
    r = O.RefAuralizer(synth, fc, N, L, backend="parallel")
    x = O.OracleAuralizer(synth, fc, N, 1, L, mu=0.0, f64=True)
    ty, tf = Tri(), Tri()
    src = noise_blocks(7, 1, N)
    for b in range(7503):
        m = next(src)
        ty.add(g.process(m), r.process(m), x.process(m))
        if b % 250 == 249 or b == 7502:
            tf.add(g.feedback_estimate()[0], r.feedback_estimate(), x.feedback_estimate()[0])
    ty.check("c3 y")
    tf.check("c3 f^")


@pytest.mark.parametrize("constrained", [False, True])
def test_c3_nlms_stream_vs_oracle(constrained):
    """configs[2] as benchmarked (NLMS mu = 0.005, lambda 0.9, the survey's
    delta = 1e-6 N): K_f + 3 = 753 blocks against the C oracle -- y every
    block, f^ every block, W after the stream; also with the constrained
    gradient (Appendix A step 2)."""
    N, L = 64, 64
    synth, fc = c3_filters()
    kw = dict(mu=0.005, lam=0.9)
    g = A.Auralizer(list(synth), list(fc), A.make_config(48000, N, 1, L),
                    afc=A.AfcParams(**kw, constrained=constrained))
    o = O.OracleAuralizer(synth, fc, N, 1, L, constrained=constrained, **kw)
    x = O.OracleAuralizer(synth, fc, N, 1, L, f64=True, constrained=constrained, **kw)
    ty, tf = Tri(), Tri()
    src = noise_blocks(7, 1, N)
    for _ in range(753):
        m = next(src)
        ty.add(g.process(m), o.process(m), x.process(m))
        tf.add(g.feedback_estimate(), o.feedback_estimate(), x.feedback_estimate())
    tag = "c3 nlms constrained" if constrained else "c3 nlms"
    ty.check(f"{tag} y")
    tf.check(f"{tag} f^")
    w_tri(g.coeffs(), o.coeffs(), x.coeffs()).check(f"{tag} W")


@pytest.mark.parametrize("N,blocks", [(64, 753), (1024, 566)])
def test_c4_mimo_nlms_stream_vs_oracle(N, blocks):
    """configs[3]: Q = P = 4 mics x 64 loudspeakers, 12 s synthesis, 1 s
    canceller per (mic, loudspeaker), NLMS on. N = 1024 streams K + 3 = 566
    blocks (every synthesis partition); N = 64 streams K_f + 3 = 753 (every
    canceller partition; the 9000-partition synthesis is covered at full
    length by the N = 1024 run and test_gpu_fullsize's impulse sweep)."""
    Q, L, n_h, n_hf = 4, 64, 576000, 48000
    rng = np.random.default_rng(4000 + N)
    synth = decaying_filters(rng, Q * L, n_h)
    fc = decaying_filters(rng, Q * L, n_hf, t60_s=0.3, scale=0.1)
    kw = dict(mu=0.005, lam=0.9)
    g = A.Auralizer(list(synth), list(fc), A.make_config(48000, N, Q, L, mimo=True), afc=A.AfcParams(**kw))
    o = O.OracleAuralizer(synth, fc, N, Q, L, **kw)
    x = O.OracleAuralizer(synth, fc, N, Q, L, f64=True, **kw)
    K = g.synth_partitions()
    assert K == -(-n_h // N)
    if N == 1024:
        assert blocks == K + 3
    ty, tf = Tri(), Tri()
    src = noise_blocks(7, Q, N)
    for b in range(blocks):
        m = next(src)
        ty.add(g.process(m), o.process(m), x.process(m))
        if b % 50 == 49 or b == blocks - 1:
            tf.add(g.feedback_estimate(), o.feedback_estimate(), x.feedback_estimate())
    ty.check(f"c4 N={N} y")
    tf.check(f"c4 N={N} f^")
    w_tri(g.coeffs(), o.coeffs(), x.coeffs()).check(f"c4 N={N} W")


C5 = dict(N=128, L=512, n_h=1920000, fs=96000, bases=4)


@pytest.fixture(scope="module")
def c5_reference():
    """configs[4] inputs and the reference's outputs for them. Loudspeaker l
    gets the DISTINCT filter base[l % 4] * (1 + l/512): its exact output is
    (1 + l/512) x the output of base[l % 4], so one reference Convolver over
    the 4 bases (parallel backend) checks all 512 channels over the whole
    stream -- a channel-mapping error shows as a scale error >= 2e-3."""
    c = C5
    rng = np.random.default_rng(5000)
    base = decaying_filters(rng, c["bases"], c["n_h"], fs=c["fs"])
    scale = (1.0 + np.arange(c["L"]) / c["L"]).astype(np.float32)
    rows = [base[l % c["bases"]] * scale[l] for l in range(c["L"])]
    ref = O.RefConvolver(base, c["N"], 1, c["bases"], O.BROADCAST, backend="parallel")
    K = ref.partitions
    assert K == 15000
    blocks = K + 3
    x = np.random.default_rng(7).standard_normal((blocks, 1, c["N"])).astype(np.float32)
    y = np.empty((blocks, c["bases"], c["N"]), np.float32)
    for b in range(blocks):
        y[b] = ref.process(x[b])
    # float64 truth: the linear convolution of the whole stream (one FFT)
    xs = x.reshape(-1).astype(np.float64)
    nfft = 1 << int(np.ceil(np.log2(xs.size + c["n_h"])))
    X = np.fft.rfft(xs, nfft)
    truth = np.stack([np.fft.irfft(X * np.fft.rfft(base[i].astype(np.float64), nfft), nfft)[:xs.size]
                      for i in range(c["bases"])]).reshape(c["bases"], blocks, c["N"]).transpose(1, 0, 2)
    return rows, scale, x, y, truth


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_c5_every_channel_full_stream(c5_reference, G):
    """configs[4] (1 x 512, 96 kHz, N = 128, 20 s): the loudspeakers split
    into G contiguous shards as the multi-GPU path does (independent
    Convolvers; here on one device), all 15003 blocks of noise input, every
    channel against the reference."""
    rows, scale, x, y, truth = c5_reference
    c = C5
    L, N, nb = c["L"], c["N"], c["bases"]
    per = L // G
    shards = [A.Convolver(rows[g * per:(g + 1) * per], A.make_config(c["fs"], N, 1, per))
              for g in range(G)]
    idx = np.arange(L) % nb
    # channel l's filter is the fp32 rounding of base * s_l: its exact output
    # is s_l x (base's) up to that one rounding per tap (~6e-8 relative)
    sc = scale.astype(np.float64)[:, None]
    t = Tri()
    for b in range(x.shape[0]):
        out = np.concatenate([s.process(x[b]) for s in shards], axis=0)
        t.add(out, sc * y[b][idx].astype(np.float64), sc * truth[b][idx])
    for s in shards:
        s.close()
    t.check(f"c5 G={G}")
