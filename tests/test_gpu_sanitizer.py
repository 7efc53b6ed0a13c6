"""GPU: compute-sanitizer (memcheck, racecheck, synccheck) over every kernel
of the product on smoke-sized engines (tests/sanitize_workload.py): graph and
stream launch modes, the fused and separate canceller heads, MIMO, virtual
shards and the measurement relaunches. Zero reported errors required; the
reports go to gpurun_out/sanitizer_<tool>.log when run on the GPU box.

racecheck excludes k_back: its shared-memory ring is filled by cp.async.bulk
(TMA) and handed between the producer lane and the consumer warps through
mbarrier expect_tx / complete_tx / try_wait, which racecheck (CUDA 12.9)
does not model -- it reports every TMA write vs the consumers' reads of the
same stage, and the producer's stage-metadata store vs their reads, as
hazards (profiles/r2_sanitizer.md keeps that log). k_back still runs under
memcheck and synccheck, and its named-barrier reduction (team_partial) is
the only shared memory it shares without an mbarrier."""
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
    if tool == "racecheck":
        cmd[3:3] = ["--kernel-name-exclude", "kns=k_backILi"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    text = open(log).read() if os.path.exists(log) else ""
    assert r.returncode == 0, (r.returncode, r.stdout[-2000:], r.stderr[-2000:], text[-4000:])
    assert "sanitize workload: ok" in r.stdout
    assert "ERROR SUMMARY: 0 errors" in text or "RACECHECK SUMMARY: 0 hazards" in text, text[-2000:]
