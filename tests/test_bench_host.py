"""CPU checks of bench.py's host logic: the lazily generated per-shard
filter rows and the weak/strong sharding of a configuration."""
import numpy as np

import bench
from paper_2509_04390_b200 import shard as S


def test_lazy_rows_are_deterministic_and_normalised():
    rows = bench.LazyRows(6, 4800, 48000, seed=11)
    assert len(rows) == 6
    a, b = rows[3], rows[3]
    assert a.dtype == np.float32 and a.shape == (4800,)
    assert np.array_equal(a, b)
    assert not np.array_equal(rows[2], rows[3])
    assert abs(float(np.dot(a.astype(np.float64), a)) - 1.0) < 1e-5
    # the -60 dB envelope: the tail is ~1e-3 of the head
    assert np.std(a[-480:]) < 0.01 * np.std(a[:480])


def test_shard_slices_of_lazy_rows_match_the_full_set():
    Q, L = 2, 8
    rows = bench.LazyRows(Q * L, 256, 48000, seed=3)
    for world in (2, 4):
        for rank in range(world):
            l0, l1 = S.shard_range(L, world, rank)
            part = S.shard_rows(rows, Q, L, l0, l1)
            want = [rows[q * L + l] for q in range(Q) for l in range(l0, l1)]
            assert all(np.array_equal(x, y) for x, y in zip(part, want))


def test_sharded_cfg_weak_and_strong():
    c3 = bench.CONFIGS["c3"]
    assert bench.sharded_cfg(c3, 1, "weak")["L"] == 64
    w = bench.sharded_cfg(c3, 8, "weak")
    assert w["L"] == 512 and "weak scaling" in w["desc"] and w["n_h"] == c3["n_h"]
    assert bench.sharded_cfg(c3, 8, "strong")["L"] == 64


def test_cpu_sample_channels_bounds_the_reference_setup():
    assert bench.cpu_sample_channels(bench.CONFIGS["c3"]) == (None, 1.0)
    L_sub, scale = bench.cpu_sample_channels(bench.CONFIGS["c5"])
    assert 1 <= L_sub < 512 and abs(scale - 512 / L_sub) < 1e-12


def test_sweep_csv_keeps_the_reference_header_and_number_format():
    """tools/sweep_csv.py extends the reference's CSV (bench.hpp:296-316);
    its first ten columns are the header test_bench.cpp:148-151 pins."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "sweep_csv", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "tools", "sweep_csv.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    assert m.HEADER == "subject,backend,parameter,value,mean_s,min_s,max_s,trials,budget_s,realtime"
    assert m.fmt(32) == "32" and m.fmt(0.25) == "0.25" and m.fmt(0.001) == "0.001"
    assert float(m.fmt(1 / 3)) == 1 / 3  # shortest round-trippable
    # filter_length_s overrides the synthesis length (bench.hpp detail::resolve)
    N, C, n_h, n_hf, fs = m.resolve("filter_length_s", 2.0)
    assert (N, C, n_h, n_hf, fs) == (128, 32, 96000, 48000, 48000)
    assert m.resolve("block_size", 64)[0] == 64 and m.resolve("channels", 8)[1] == 8
