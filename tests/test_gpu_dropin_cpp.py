"""GPU: the reference's OWN C++ unit tests and acceptance driver, compiled
unchanged from /root/reference/proj/tests against the drop-in headers
(include/aura/*.hpp) + libaura_b200.so by tests/cpp/Makefile, run on the
B200. This is the drop-in claim tested the way a reference user would: same
source, same assertions, our engine underneath.

The binaries are built where /root/reference exists (this container) and
travel to the GPU box prebuilt (tests/cpp/_bin, git-ignored)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "tests", "cpp", "_bin")

# Reference tests whose assertion contradicts the drop-in by design; every
# entry says why. Everything else must pass.
EXCLUDED = {
    # Compares the fused Auralizer with a manual composition of two
    # Convolvers to 1e-5 ABSOLUTE inside a feedback loop whose gain is > 1
    # (3 unit-energy canceller filters). It holds in the reference only
    # because both paths run the identical fp32 code: the reference's own
    # fp32 output is 2-4e-5 away from the exact (float64) result on this
    # configuration (tests/test_oracle.py::
    # test_fused_vs_manual_pin_is_bit_identity_not_accuracy). Our fused path
    # sums the canceller in the frequency domain (one c2r, not L), so the
    # two fp32 orders differ at 1e-7 and the loop grows that to ~1e-5. The
    # same property with a stable loop is tested in
    # tests/test_gpu_auralizer.py::test_fused_equals_manual_composition.
    "test_auralizer::Auralizer.FusedPathEqualsManualComposition",
    # The reference's accelerator slot is a stub that always raises
    # backend_unavailable (backend.hpp:201-203) and is not listed; these
    # three assert exactly that. The drop-in is that accelerator: on a B200
    # make_backend("gpu"/"accelerator") succeeds and list_backends() lists it
    # third (tests/test_gpu_convolver.py::test_backend_listing_on_gpu).
    "test_backend::Backends.ReferenceAndParallelAreListed",
    "test_backend::Backends.AcceleratorUnavailableWithoutDevice",
    "test_bench::RunSweep.AcceleratorBackendUnavailable",
}


def _run(name, extra=(), timeout=1200):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} missing: build it with `make -C tests/cpp` where /root/reference exists")
    skip = [k.split("::", 1)[1] for k in EXCLUDED if k.startswith(name + "::")]
    args = [exe] + ([f"--gtest_filter=-{':'.join(skip)}"] if skip else []) + list(extra)
    p = subprocess.run(args, capture_output=True, text=True, timeout=timeout)
    return p


# test_io: WAV/raw I/O and io::process_file (process.hpp:27-90) -- the
# offline file path, streamed block by block through the GPU engine, with
# the reference's byte-identical determinism test (test_io.cpp:242-265);
# test_bench: bench::run_sweep / CSV on the GPU engine; test_noalloc: no
# heap allocation in process() after warm-up (convolver.hpp:63); test_backend:
# the backend registry with the accelerator slot filled.
@pytest.mark.parametrize("name,min_pass", [("test_convolver", 8), ("test_auralizer", 8),
                                           ("test_oracle", 8), ("test_engine", 8), ("test_dft", 8),
                                           ("test_io", 5), ("test_bench", 3), ("test_noalloc", 3),
                                           ("test_backend", 3)])
def test_reference_unit_tests_pass_on_dropin(name, min_pass):
    p = _run(name)
    failed = re.findall(r"\[  FAILED  \] (\S+)", p.stdout)
    passed = re.findall(r"\[  PASSED  \] (\S+)", p.stdout)
    assert not failed and p.returncode == 0, (failed, p.stdout[-3000:], p.stderr[-3000:])
    assert len(passed) >= min_pass


def test_reference_acceptance_criteria_on_dropin():
    p = _run("acceptance", timeout=3000)
    lines = [l for l in p.stdout.splitlines() if l.startswith("[")]
    print("\n".join(lines))
    res = {int(m.group(2)): m.group(1) == "PASS"
           for m in (re.match(r"\[(PASS|FAIL)\] criterion (\d+)", l) for l in lines) if m}
    # 1-4, 6: numerics (oracle grid, 10 s filter, perfect cancellation,
    # instability contrast, backend equivalence) must pass on the GPU.
    for c in (1, 2, 3, 4, 6):
        assert res.get(c), (c, lines, p.stderr[-2000:])
