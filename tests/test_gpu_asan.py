"""GPU: the host side of the C-ABI (engine construction, planner, graph
capture, process / shard / measurement entry points, error paths) under
AddressSanitizer + UndefinedBehaviorSanitizer. The same smoke
workload as the compute-sanitizer test runs against libaura_b200_asan.so
(`make -C paper_2509_04390_b200 asan`, built on demand) with libasan
preloaded; any ASan report or UBSan runtime error fails the test."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2509_04390_b200")
LIB = os.path.join(PKG, "libaura_b200_asan.so")


def _libasan():
    out = subprocess.run(["gcc", "-print-file-name=libasan.so"], capture_output=True, text=True)
    path = out.stdout.strip()
    return path if os.path.isabs(path) and os.path.exists(path) else None


def test_host_side_asan_ubsan_clean():
    asan = _libasan()
    if asan is None:
        pytest.skip("libasan not available")
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", PKG, "asan"], check=True, timeout=900)
    env = dict(os.environ)
    env.update({
        "LD_PRELOAD": asan,
        # the CUDA driver maps memory inside ASan's shadow gap; Python's own
        # allocator leaks by design at exit
        "ASAN_OPTIONS": "protect_shadow_gap=0:detect_leaks=0:halt_on_error=1",
        "UBSAN_OPTIONS": "halt_on_error=1:print_stacktrace=1",
        "AURA_B200_LIB": LIB,
    })
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_workload.py")],
                       env=env, capture_output=True, text=True, timeout=1200)
    with open(os.path.join(out_dir, "asan_ubsan.log"), "w") as f:
        f.write(r.stdout + "\n" + r.stderr)
    bad = [ln for ln in r.stderr.splitlines() if "AddressSanitizer" in ln or "runtime error:" in ln]
    assert r.returncode == 0 and not bad, (r.returncode, bad[:5], r.stderr[-2000:])
    assert "sanitize workload: ok" in r.stdout
    assert f"library: {LIB}" in r.stdout  # the instrumented build ran
