"""CPU: the product C-ABI library loads, exports every symbol declared in
include/aura_b200.h (the drop-in boundary) and include/aura_b200_diag.h
(measurement), and -- with no B200 present -- fails loudly instead of
falling back to a CPU path."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2509_04390_b200 as A
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "aura_b200.h")
DIAG = os.path.join(ROOT, "include", "aura_b200_diag.h")


def declared_symbols(path=HEADER):
    text = open(path).read()
    # declarations only: "<type> aura_b200_x(" at the start of a line
    return sorted(set(re.findall(r"^[a-z][\w *]*?\b(aura_b200_[a-z_0-9]+)\s*\(", text, re.M)))


def test_library_built_and_loads():
    assert os.path.exists(A.LIB_PATH), "run __graft_entry__.build()"
    assert A.lib().aura_b200_abi_version() == 2


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    diag = declared_symbols(DIAG)
    assert len(syms) >= 22 and len(diag) >= 10
    assert not set(syms) & set(diag)
    lib = C.CDLL(A.LIB_PATH)
    missing = [s for s in syms + diag if not hasattr(lib, s)]
    assert not missing, missing


def test_error_codes_mirror_reference_enum():
    # engine.hpp:15-37 order; the C-ABI returns 1 + code
    text = open(HEADER).read()
    m = dict(re.findall(r"AURA_B200_E_([A-Z_]+) = (\d+)", text))
    for code in A.ErrorCode:
        if code.value <= A.ErrorCode.invalid_argument:
            assert int(m[code.name.upper()]) == code.value + 1


def test_config_validation_matches_reference():
    # test_engine.cpp:23-73 error codes
    cases = [((0, 64, 1, 1), A.ErrorCode.zero_sample_rate),
             ((48000, 48, 1, 1), A.ErrorCode.non_power_of_two_block),
             ((48000, 8, 1, 1), A.ErrorCode.non_power_of_two_block),
             ((48000, 16384, 1, 1), A.ErrorCode.non_power_of_two_block),
             ((48000, 64, 2, 3), A.ErrorCode.bad_channel_combination),
             ((48000, 64, 1, 0), A.ErrorCode.bad_channel_combination)]
    for args, code in cases:
        with pytest.raises(A.Error) as ei:
            A.make_config(*args)
        assert ei.value.code == code
    cfg = A.make_config(48000, 128, 1, 32)
    assert cfg.fft_size == 256 and cfg.bins() == 129
    assert A.latency_budget(A.make_config(48000, 64, 1, 1)) == pytest.approx(64 / 48000)
    bad = A.EngineConfig(48000, 64, 100, 1, 1)
    with pytest.raises(A.Error) as ei:
        A.validate_config(bad)
    assert ei.value.code == A.ErrorCode.fft_size_mismatch


def test_filter_errors_before_device():
    cfg = A.make_config(48000, 64, 1, 2)
    with pytest.raises(A.Error) as ei:
        A.Convolver([np.ones(100), np.ones(200)], cfg)
    assert ei.value.code == A.ErrorCode.filter_length_mismatch
    with pytest.raises(A.Error) as ei:
        A.Convolver([], cfg)
    assert ei.value.code == A.ErrorCode.empty_filter
    with pytest.raises(A.Error) as ei:
        A.Convolver([np.zeros(0)], A.make_config(48000, 64, 1, 1))
    assert ei.value.code == A.ErrorCode.empty_filter
    with pytest.raises(A.Error) as ei:
        A.Auralizer([np.ones(4)] * 4, [np.ones(4)] * 2, A.make_config(48000, 64, 1, 4))
    assert ei.value.code == A.ErrorCode.channel_count_mismatch


def test_cpu_backends_are_not_offered():
    for name in ("reference", "parallel", "cpu", "bogus"):
        with pytest.raises(A.Error) as ei:
            A.make_backend(name)
        assert ei.value.code == A.ErrorCode.backend_unavailable


def _no_gpu():
    n = C.c_int(-1)
    A.lib().aura_b200_device_count(C.byref(n))
    return n.value == 0


@pytest.mark.skipif(not _no_gpu(), reason="a B200 is present")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(A.Error) as ei:
        A.Convolver([np.ones(10, np.float32)], A.make_config(48000, 64, 1, 1))
    assert ei.value.code == A.ErrorCode.backend_unavailable
    assert A.list_backends() == []
    with pytest.raises(A.Error) as ei:
        A.make_backend("gpu")
    assert ei.value.code == A.ErrorCode.backend_unavailable
