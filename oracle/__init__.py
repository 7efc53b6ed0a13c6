"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the parity checker.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2509_04390_b200``) never imports it.

Two checkers live here:

* ``Oracle*`` wrap ``liboracle.so``: the plain-C restatement of the
  reference hot path (``oracle/aura_oracle.c``), extended with the
  Appendix-A NLMS update and Appendix-B MIMO composition. ``f64=True``
  selects ``liboracle64.so``, the same algorithm in float64 with exact
  twiddles: the ground truth for full-length streams, where every fp32
  implementation (the reference included) drifts ~1e-5 of the RMS.
* ``Ref*`` wrap ``_ref/libaura_ref.so``: the unmodified reference headers
  (``/root/reference/proj/include/aura``) behind a C shim
  (``oracle/ref_shim.cpp``), built with the reference's Release flags.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(HERE, "liboracle.so")
_ORACLE64_SO = os.path.join(HERE, "liboracle64.so")
_REF_SO = os.path.join(HERE, "_ref", "libaura_ref.so")

BROADCAST, ELEMENTWISE, MIMO = 0, 1, 2

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_olib = {}
_rlib = None


def olib(f64=False):
    if f64 not in _olib:
        L = _load(_ORACLE64_SO if f64 else _ORACLE_SO)
        _f32p = _f64p if f64 else globals()["_f32p"]
        C_real = C.c_double if f64 else C.c_float
        L.ao_plan_new.restype = C.c_void_p
        L.ao_plan_new.argtypes = [_sz]
        L.ao_plan_free.argtypes = [C.c_void_p]
        L.ao_forward.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ao_inverse.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ao_conv_new.restype = C.c_void_p
        L.ao_conv_new.argtypes = [_sz, _sz, _sz, C.c_int, _f32p, _sz]
        L.ao_conv_free.argtypes = [C.c_void_p]
        L.ao_conv_process.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ao_conv_reset.argtypes = [C.c_void_p]
        L.ao_conv_partitions.restype = _sz
        L.ao_conv_partitions.argtypes = [C.c_void_p]
        L.ao_conv_spectrum.argtypes = [C.c_void_p, _sz, _sz, _f32p]
        L.ao_aur_new.restype = C.c_void_p
        L.ao_aur_new.argtypes = [_sz, _sz, _sz, _f32p, _sz, _f32p, _sz,
                                 C_real, C_real, C_real, C_real]
        L.ao_aur_free.argtypes = [C.c_void_p]
        L.ao_aur_process.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ao_aur_reset.argtypes = [C.c_void_p]
        L.ao_aur_set_gain.argtypes = [C.c_void_p, C_real]
        L.ao_aur_set_constrained.argtypes = [C.c_void_p, C.c_int]
        L.ao_aur_set_constrained.restype = C.c_int
        L.ao_aur_feedback_estimate.argtypes = [C.c_void_p, _f32p]
        L.ao_aur_fc_partitions.restype = _sz
        L.ao_aur_fc_partitions.argtypes = [C.c_void_p]
        L.ao_aur_synth_partitions.restype = _sz
        L.ao_aur_synth_partitions.argtypes = [C.c_void_p]
        L.ao_aur_coeffs.argtypes = [C.c_void_p, _f32p]
        L.ao_aur_power.argtypes = [C.c_void_p, _f32p]
        L.ao_direct_convolve.argtypes = [_f64p, _sz, _f64p, _sz, _f64p]
        _olib[f64] = L
    return _olib[f64]


def ref_available() -> bool:
    return os.path.exists(_REF_SO) or os.path.isdir("/root/reference/proj/include/aura")


def rlib():
    global _rlib
    if _rlib is None:
        L = _load(_REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_conv_new.argtypes = [_sz, _sz, _sz, C.c_int, _f32p, _sz, _sz,
                                   C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_conv_process.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ref_conv_reset.argtypes = [C.c_void_p]
        L.ref_conv_partitions.restype = _sz
        L.ref_conv_partitions.argtypes = [C.c_void_p]
        L.ref_conv_spectrum.argtypes = [C.c_void_p, _sz, _sz, _f32p]
        L.ref_conv_free.argtypes = [C.c_void_p]
        L.ref_aur_new.argtypes = [_sz, _sz, _f32p, _sz, _f32p, _sz, C.c_float,
                                  C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_aur_process.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ref_aur_estimate.argtypes = [C.c_void_p, _f32p]
        L.ref_aur_reset.argtypes = [C.c_void_p]
        L.ref_aur_free.argtypes = [C.c_void_p]
        L.ref_forward.argtypes = [_sz, _f32p, _f32p]
        L.ref_inverse.argtypes = [_sz, _f32p, _f32p]
        L.ref_direct_convolve.argtypes = [_f64p, _sz, _f64p, _sz, _f64p]
        L.ref_partition_count.restype = _sz
        L.ref_partition_count.argtypes = [_sz, _sz]
        L.ref_backend_workers.restype = C.c_uint
        L.ref_backend_workers.argtypes = [C.c_char_p]
        L.ref_verify.argtypes = [C.c_int, C.c_char_p, _sz]
        _rlib = L
    return _rlib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- oracle


def forward(buf: np.ndarray) -> np.ndarray:
    """r2c of len n_f -> (n_f/2+1) complex64 (dft.hpp:69-101)."""
    buf = _f32(buf)
    p = olib().ao_plan_new(buf.size)
    out = np.zeros(buf.size + 2, np.float32)
    olib().ao_forward(p, buf, out)
    olib().ao_plan_free(p)
    return out.view(np.complex64)


def inverse(spec: np.ndarray) -> np.ndarray:
    spec = np.ascontiguousarray(spec, dtype=np.complex64)
    n_f = 2 * (spec.size - 1)
    p = olib().ao_plan_new(n_f)
    out = np.zeros(n_f, np.float32)
    olib().ao_inverse(p, spec.view(np.float32), out)
    olib().ao_plan_free(p)
    return out


def direct_convolve(x, h) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    h = np.ascontiguousarray(h, np.float64)
    y = np.zeros(x.size + h.size - 1, np.float64)
    olib().ao_direct_convolve(x, x.size, h, h.size, y)
    return y


class OracleConvolver:
    """CPU restatement of aura::Convolver (convolver.hpp:65-220).

    filters: (rows, n_h). mode BROADCAST (inputs=1), ELEMENTWISE
    (inputs=outputs) or MIMO (rows = inputs*outputs, row q*L+l).
    f64: the float64 ground-truth build (inputs are the same float32
    values, exactly widened; outputs float64)."""

    def __init__(self, filters, block, inputs, outputs, mode, f64=False):
        self.f64 = f64
        self.dt = np.float64 if f64 else np.float32
        f = np.ascontiguousarray(_f32(filters), self.dt)
        self.N, self.inputs, self.outputs = block, inputs, outputs
        self._L = olib(f64)
        self._h = self._L.ao_conv_new(block, inputs, outputs, mode, f, f.shape[1])
        if not self._h:
            raise ValueError("oracle rejected the convolver configuration")
        self.partitions = self._L.ao_conv_partitions(self._h)

    def process(self, x):
        x = np.ascontiguousarray(_f32(x), self.dt).reshape(self.inputs, self.N)
        out = np.zeros((self.outputs, self.N), self.dt)
        self._L.ao_conv_process(self._h, x, out)
        return out

    def reset(self):
        self._L.ao_conv_reset(self._h)

    def spectrum(self, row, k):
        out = np.zeros(2 * (self.N + 1), self.dt)
        self._L.ao_conv_spectrum(self._h, row, k, out)
        return out.view(np.complex128 if self.f64 else np.complex64)

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ao_conv_free(self._h)
            self._h = None


class OracleAuralizer:
    """CPU restatement of aura::Auralizer (auralizer.hpp:25-123) plus the
    SURVEY Appendix-A NLMS update (mu > 0) and Appendix-B MIMO (inputs>1).
    synth: (Q*L, n_h); fc: (P*L, n_hf) with P = Q."""

    def __init__(self, synth, fc, block, inputs, outputs, gain=1.0, mu=0.0,
                 lam=0.9, delta=None, f64=False, constrained=False):
        self.f64 = f64
        self.dt = np.float64 if f64 else np.float32
        s = np.ascontiguousarray(_f32(synth), self.dt)
        f = np.ascontiguousarray(_f32(fc), self.dt)
        if delta is None:
            delta = 1e-6 * block  # same default as the product
        # the parameters as the fp32 engines hold them (exactly widened in f64)
        gain, mu, lam, delta = (float(np.float32(v)) for v in (gain, mu, lam, delta))
        self.N, self.Q, self.L = block, inputs, outputs
        self._L = olib(f64)
        self._h = self._L.ao_aur_new(block, inputs, outputs, s, s.shape[1], f,
                                     f.shape[1], gain, mu, lam, delta)
        if not self._h:
            raise ValueError("oracle rejected the auralizer configuration")
        self.fc_partitions = self._L.ao_aur_fc_partitions(self._h)
        self.synth_partitions = self._L.ao_aur_synth_partitions(self._h)
        if constrained and self._L.ao_aur_set_constrained(self._h, 1) != 0:
            raise MemoryError("oracle: constrained-update scratch")

    def process(self, mic):
        mic = np.ascontiguousarray(_f32(mic), self.dt).reshape(self.Q, self.N)
        out = np.zeros((self.L, self.N), self.dt)
        self._L.ao_aur_process(self._h, mic, out)
        return out

    def reset(self):
        self._L.ao_aur_reset(self._h)

    def set_gain(self, g):
        self._L.ao_aur_set_gain(self._h, float(np.float32(g)))

    def feedback_estimate(self):
        out = np.zeros((self.Q, self.N), self.dt)
        self._L.ao_aur_feedback_estimate(self._h, out)
        return out

    def coeffs(self):
        out = np.zeros(self.Q * self.L * self.fc_partitions * (self.N + 1) * 2, self.dt)
        self._L.ao_aur_coeffs(self._h, out)
        return out.view(np.complex128 if self.f64 else np.complex64).reshape(
            self.Q, self.L, self.fc_partitions, self.N + 1)

    def power(self):
        out = np.zeros(self.N + 1, self.dt)
        self._L.ao_aur_power(self._h, out)
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ao_aur_free(self._h)
            self._h = None


# ------------------------------------------------------------- reference


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code  # 1 + aura::ErrorCode


def _rcheck(rc):
    if rc:
        raise RefError(rc, rlib().ref_last_error().decode())


class RefConvolver:
    """The unmodified reference aura::Convolver via oracle/_ref."""

    def __init__(self, filters, block, inputs, outputs, mode, backend="reference"):
        f = _f32(filters)
        self.N, self.inputs, self.outputs = block, inputs, outputs
        h = C.c_void_p()
        _rcheck(rlib().ref_conv_new(block, inputs, outputs, mode, f, f.shape[0],
                                    f.shape[1], backend.encode(), C.byref(h)))
        self._h = h
        self.partitions = rlib().ref_conv_partitions(h)

    def process(self, x):
        x = _f32(x).reshape(self.inputs, self.N)
        out = np.zeros((self.outputs, self.N), np.float32)
        _rcheck(rlib().ref_conv_process(self._h, x, out))
        return out

    def reset(self):
        rlib().ref_conv_reset(self._h)

    def spectrum(self, c, k):
        out = np.zeros(2 * (self.N + 1), np.float32)
        rlib().ref_conv_spectrum(self._h, c, k, out)
        return out.view(np.complex64)

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().ref_conv_free(self._h)
            self._h = None


class RefAuralizer:
    """The unmodified reference aura::Auralizer via oracle/_ref."""

    def __init__(self, synth, fc, block, outputs, gain=1.0, backend="reference"):
        s, f = _f32(synth), _f32(fc)
        self.N, self.L = block, outputs
        h = C.c_void_p()
        _rcheck(rlib().ref_aur_new(block, outputs, s, s.shape[1], f, f.shape[1],
                                   gain, backend.encode(), C.byref(h)))
        self._h = h

    def process(self, mic):
        mic = _f32(mic).reshape(1, self.N)
        out = np.zeros((self.L, self.N), np.float32)
        _rcheck(rlib().ref_aur_process(self._h, mic, out))
        return out

    def feedback_estimate(self):
        out = np.zeros(self.N, np.float32)
        rlib().ref_aur_estimate(self._h, out)
        return out

    def reset(self):
        rlib().ref_aur_reset(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().ref_aur_free(self._h)
            self._h = None


def ref_forward(buf):
    buf = _f32(buf)
    out = np.zeros(buf.size + 2, np.float32)
    _rcheck(rlib().ref_forward(buf.size, buf, out))
    return out.view(np.complex64)


def ref_inverse(spec):
    spec = np.ascontiguousarray(spec, dtype=np.complex64)
    n_f = 2 * (spec.size - 1)
    out = np.zeros(n_f, np.float32)
    _rcheck(rlib().ref_inverse(n_f, spec.view(np.float32), out))
    return out


def ref_direct_convolve(x, h):
    x = np.ascontiguousarray(x, np.float64)
    h = np.ascontiguousarray(h, np.float64)
    y = np.zeros(x.size + h.size - 1, np.float64)
    rlib().ref_direct_convolve(x, x.size, h, h.size, y)
    return y


def ref_backend_workers(name="parallel") -> int:
    return int(rlib().ref_backend_workers(name.encode()))


def ref_verify(full=False):
    buf = C.create_string_buffer(1 << 20)
    rc = rlib().ref_verify(1 if full else 0, buf, len(buf))
    return rc == 0, buf.value.decode()
