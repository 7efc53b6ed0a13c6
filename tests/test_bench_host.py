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


def test_gpus_flag_relaunches_one_process_per_rank():
    """`bench.py --gpus 2` without torchrun re-launches itself under
    torch.distributed.run; the reference arm runs on rank 0 only and prints
    ONE line whose n_gpus is the requested world (CPU-only: the reference arm
    needs no GPU)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 3
    assert "weak scaling" in d["config"]["workload"]


def test_l2_roofline_peak_from_the_committed_probe():
    peak, kind = bench.l2_read_peak(64e6)
    assert peak is not None and 5000 < peak < 20000 and "r2_l2_probe" in kind
    assert bench.roofline_regime(65.3e6) == "l2" and bench.roofline_regime(323e6) == "hbm"
