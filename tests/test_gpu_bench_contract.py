"""GPU: bench.py's JSON line keeps the driver contract (one line, the
BASELINE metric, value / e2e / roofline / cpu_baseline / clocks /
gpu_launches / max_realtime keys) on a short run."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_line_contract():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3",
                          "--max-rt-s", "20", "--cpu-blocks", "3"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["metric"].startswith("per-block latency p50/p99") and d["unit"] == "us"
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3
    assert d["higher_is_better"] is False and d["dtype"] == "f32"
    assert 0 < d["p50_us"] <= d["value"] < d["budget_us"]
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == 4 * 64 and e2e["d2h_bytes_per_step"] == 4 * 64 * 64
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.5 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    cpu = d["cpu_baseline"]
    assert cpu["kind"] == "reference" and cpu["cores"] >= 1 and cpu["value"] > d["value"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["gpu_launches"] == 20 * 3  # k_front, k_back, k_reduce per block
    m = d["max_realtime"]
    assert m["channels"] >= 64 and m["channels_x_taps"] == m["channels"] * 480000
    assert d["c5"]["realtime"] is True
