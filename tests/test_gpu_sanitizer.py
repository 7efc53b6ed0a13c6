"""GPU: compute-sanitizer (memcheck, racecheck, synccheck) over every kernel
of the product on smoke-sized engines (tests/sanitize_workload.py): graph and
stream launch modes, the fused and separate canceller heads, MIMO, virtual
shards and the measurement relaunches. Zero reported errors required; the
reports go to gpurun_out/sanitizer_<tool>.log when run on the GPU box."""
import os
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    pytest.fail("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    log = os.path.join(out_dir, f"sanitizer_{tool}.log")
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "99", "--log-file", log,
           sys.executable, os.path.join(ROOT, "tests", "sanitize_workload.py")]
    if tool == "memcheck":
        cmd[3:3] = ["--leak-check", "no"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    text = open(log).read() if os.path.exists(log) else ""
    assert r.returncode == 0, (r.returncode, r.stdout[-2000:], r.stderr[-2000:], text[-4000:])
    assert "sanitize workload: ok" in r.stdout
    assert "ERROR SUMMARY: 0 errors" in text or "RACECHECK SUMMARY: 0 hazards" in text, text[-2000:]
