"""GPU: engine robustness -- the 64-bit block counter across 2^32, the
shard-exchange timeout path, and measurement calls that must leave the
canceller state untouched."""
import numpy as np
import pytest

import paper_2509_04390_b200 as A
from paper_2509_04390_b200 import shard as S
from conftest import decaying_filters

pytestmark = pytest.mark.gpu


def small_aur(mu=0.02, N=64, L=8, seed=3):
    rng = np.random.default_rng(seed)
    synth = decaying_filters(rng, L, 9 * N + 5, scale=0.5)
    fc = decaying_filters(rng, L, 3 * N + 1, scale=0.1)
    mk = lambda: A.Auralizer(list(synth), list(fc), A.make_config(48000, N, 1, L),
                             input_gain=0.9, afc=A.AfcParams(mu, 0.9, 1e-2))
    return mk, rng


@pytest.mark.parametrize("mu", [0.0, 0.02])
def test_block_counter_crosses_2_32(mu):
    """A 32-bit block counter wraps after 2^32 blocks (16.6 days at N = 16)
    and, as 2^32 is no multiple of K, reorders every delay-line ring at the
    wrap. Numbered from 2^32 - 5, an engine must stream bit-identically to
    a fresh one across the boundary (ring slots are block mod K)."""
    mk, rng = small_aur(mu)
    fresh, seeked = mk(), mk()
    seeked.seek_block(2**32 - 5)
    for b in range(30):
        m = rng.standard_normal((1, 64)).astype(np.float32)
        assert np.array_equal(fresh.process(m), seeked.process(m)), b
        assert np.array_equal(fresh.feedback_estimate(), seeked.feedback_estimate()), b
    for age in (0, 3, 9):
        assert np.array_equal(fresh.fdl_slot(0, 0, age), seeked.fdl_slot(0, 0, age))
        assert np.array_equal(fresh.fdl_slot(1, 5, min(age, 3)), seeked.fdl_slot(1, 5, min(age, 3)))
    assert np.array_equal(fresh.coeffs(), seeked.coeffs())
    with pytest.raises(A.Error):
        seeked.seek_block(7)  # only before the first block
    seeked.reset()
    seeked.seek_block(2**40 + 3)


def test_time_phase_leaves_engine_state_untouched():
    """time_phase relaunches single kernels for the roofline timing -- k_back
    applies the NLMS update in place, k_reduce advances the block, the fused
    canceller head shifts the loudspeaker history: W and every later output
    must be exactly as if it had never run."""
    mk, rng = small_aur(0.02)
    a, b = mk(), mk()
    mics = rng.standard_normal((20, 1, 64)).astype(np.float32)
    for i in range(10):
        a.process(mics[i])
        b.process(mics[i])
    a.synchronize()
    W = a.coeffs().copy()
    a.time_phase("k_back", 7)
    a.time_phase("k_reduce", 5)
    a.time_phase("k_front", 5)
    assert np.array_equal(a.coeffs(), W)
    for i in range(10, 20):
        assert np.array_equal(a.process(mics[i]), b.process(mics[i]))
    assert np.array_equal(a.coeffs(), b.coeffs())


def test_shard_exchange_timeout_reports_and_reset_recovers():
    """A shard whose peer never delivers its canceller partial waits 5 s
    (bounded, never a hung GPU), keeps its previous f^ instead of summing
    stale slots, and fails every call with TIMEOUT until a coordinated
    reset of all shards."""
    N, L = 64, 8
    rng = np.random.default_rng(9)
    synth = decaying_filters(rng, L, 9 * N, scale=0.5)
    fc = decaying_filters(rng, L, 3 * N, scale=0.1)
    cfg = A.make_config(48000, N, 1, L)
    afc = A.AfcParams(0.02, 0.9, 1e-2)
    v = S.VirtualShards(list(synth), list(fc), cfg, 2, afc=afc)
    ref = S.VirtualShards(list(synth), list(fc), cfg, 2, afc=afc)
    m = rng.standard_normal((1, N)).astype(np.float32)
    v.shards[0].process(m)  # shard 1 never runs this block
    with pytest.raises(A.Error) as ei:
        v.shards[0].synchronize()
    assert ei.value.code == A.ErrorCode.timeout
    with pytest.raises(A.Error):
        v.shards[0].process(m)
    for s in v.shards:
        s.reset()
    mics = rng.standard_normal((12, 1, N)).astype(np.float32)
    for i in range(12):
        assert np.array_equal(v.process(mics[i]), ref.process(mics[i]))
    ests = v.feedback_estimates()
    assert np.array_equal(ests[0], ests[1])
    v.close()
    ref.close()


def test_canceller_checkpoint_resumes_bit_identically():
    """afc_coeffs / afc_load_coeffs as a checkpoint of the NLMS canceller:
    an engine whose W is loaded from another's is bit-identical to an engine
    created with those spectra's filters when both start fresh (W at load =
    the partitioned F^), and an exported W loaded back continues exactly."""
    N, L = 64, 8
    rng = np.random.default_rng(31)
    synth = decaying_filters(rng, L, 9 * N, scale=0.5)
    fc_a = decaying_filters(rng, L, 3 * N, scale=0.1)
    fc_b = decaying_filters(rng, L, 3 * N, scale=0.1)
    cfg = A.make_config(48000, N, 1, L)
    afc = A.AfcParams(0.02, 0.9, 1e-2)
    a = A.Auralizer(list(synth), list(fc_a), cfg, afc=afc)
    b = A.Auralizer(list(synth), list(fc_b), cfg, afc=afc)
    b.load_coeffs(a.coeffs(), as_initial=True)   # b now starts from F^_a
    mics = rng.standard_normal((20, 1, N)).astype(np.float32)
    for i in range(20):
        assert np.array_equal(a.process(mics[i]), b.process(mics[i])), i
    assert np.array_equal(a.coeffs(), b.coeffs())
    b.reset()  # back to the loaded spectra (as_initial)
    a.reset()
    for i in range(5):
        assert np.array_equal(a.process(mics[i]), b.process(mics[i]))
    W = a.coeffs()
    W[0, 0, 0, 0] = W[0, 0, 0, 0] + 1j  # DC must be real
    with pytest.raises(A.Error) as ei:
        b.load_coeffs(W)
    assert ei.value.code == A.ErrorCode.non_real_edge_bins


def test_measurement_entry_points_run_and_leave_the_stream_consistent():
    """The diag.cu entry points bench.py and tools/ use: device-resident and
    host-I/O traced timelines, the span timing, per-phase timing -- and the
    engine still streams bit-identically to an untouched twin afterwards
    (they advance the block counter, which only moves ring slots)."""
    mk, rng = small_aur(0.02)
    a, b = mk(), mk()
    mics = rng.standard_normal((8, 1, 64)).astype(np.float32)
    tr = a.trace_blocks(6)
    trh = a.trace_blocks(6, host_inputs=mics)
    for t in (tr, trh):
        assert {"k_front", "k_back", "k_reduce", "output", "cycle"} <= set(t)
        assert np.all(t["output"][:, 0] > 0) and np.all(t["cycle"][:, 0] > t["output"][:-1, 0])
    assert a.time_device_span(10, mics) > 0
    lat, us = a.time_device_blocks(10, mics)
    assert np.all(us > 0) and np.all(lat > 0)
    ph = a.profile_phases(3)
    assert ph["k_back"][1] > 0
    a.reset()
    b.reset()
    for i in range(8):
        assert np.array_equal(a.process(mics[i]), b.process(mics[i]))


def test_early_canceller_reduction_is_bit_identical(monkeypatch):
    """k_reduce's single canceller CTA normally starts as soon as k_back has
    published the canceller partials (afc_seq words) instead of after all of
    k_back. Same partials, same summation order: the stream must be
    bit-identical to the griddepcontrol path (AURA_B200_AFC_EARLY=0), also
    after a reset, which must clear the published words (block numbers
    restart, so stale words would otherwise match)."""
    rng = np.random.default_rng(11)
    N, L = 64, 64
    synth = decaying_filters(rng, L, 200 * N + 7, scale=0.5)
    fc = decaying_filters(rng, L, 750 * N, scale=0.1)  # c3's canceller: 48k taps, 120 partials

    def mk():
        return A.Auralizer(list(synth), list(fc), A.make_config(48000, N, 1, L), input_gain=0.9,
                           afc=A.AfcParams(0.005, 0.9, None))

    on = mk()
    monkeypatch.setenv("AURA_B200_AFC_EARLY", "0")
    off = mk()
    monkeypatch.delenv("AURA_B200_AFC_EARLY")
    assert "AFC_EARLY=0" in off.describe() and "AFC_EARLY" not in on.describe()
    mics = rng.standard_normal((40, 1, N)).astype(np.float32)
    first = []
    for b, m in enumerate(mics):
        y = on.process(m)
        assert np.array_equal(y, off.process(m)), b
        assert np.array_equal(on.feedback_estimate(), off.feedback_estimate()), b
        first.append(y)
    assert np.array_equal(on.coeffs(), off.coeffs())
    on.reset()
    for b, m in enumerate(mics):
        assert np.array_equal(on.process(m), first[b]), b


def test_zero_copy_io_matches_process():
    """aura_b200_io_buffers / process_io (the mapped staging blocks, no host
    copies) stream bit-identically to process(); a non-finite input in the
    mapped block is rejected before anything is launched."""
    mk, rng = small_aur(0.02)
    a, b = mk(), mk()
    xin, xout = b.io_buffers()
    assert xin.shape == (1, 64) and xout.shape == (8, 64)
    for blk in range(40):
        m = rng.standard_normal((1, 64)).astype(np.float32)
        y = a.process(m)
        xin[...] = m
        b.process_io()
        assert np.array_equal(y, xout), blk
    assert np.array_equal(a.feedback_estimate(), b.feedback_estimate())
    xin[0, 3] = np.nan
    with pytest.raises(A.Error) as ei:
        b.process_io()
    assert ei.value.code == A.ErrorCode.non_finite_input
    assert b.blocks_processed() == 40
    m = rng.standard_normal((1, 64)).astype(np.float32)
    xin[...] = m
    b.process_io()
    assert np.array_equal(a.process(m), xout)


def test_deadline_stats_count_budget_misses():
    """Failure detection: calls whose host-visible latency exceeds N / f_s
    are counted. At 48 kHz the 1.33 ms budget of N = 64 is (all but) never
    missed; at a
    (fictitious) 2 MHz sample rate the budget of N = 16 is 8 us, below what a
    launch plus a PCIe round trip takes, so (nearly) every call misses.
    reset() clears the statistics."""
    mk, rng = small_aur(0.02)
    a = mk()
    for _ in range(20):
        a.process(rng.standard_normal((1, 64)).astype(np.float32))
    st = a.deadline_stats()
    # (a rare host-side stall can push one call over 1.33 ms)
    assert st["misses"] <= 1 and 0 < st["last_us"] <= st["max_us"]
    assert st["misses"] == (1 if st["max_us"] > st["budget_us"] else 0)
    assert abs(st["budget_us"] - 64 / 48000 * 1e6) < 1e-6
    a.reset()
    assert a.deadline_stats()["misses"] == 0 and a.deadline_stats()["max_us"] == 0.0
    synth = [np.r_[1.0, np.zeros(200)].astype(np.float32)] * 2
    fast = A.Convolver(synth, A.make_config(2_000_000, 16, 1, 2))
    for _ in range(50):
        fast.process(np.ones((1, 16), np.float32))
    st = fast.deadline_stats()
    assert st["budget_us"] == 8.0
    assert st["misses"] >= 45 and st["max_us"] >= st["last_us"] > 0
