"""B200-native UPOLS convolver + acoustic feedback canceller.

Python mirror of the reference's C++ API (``/root/reference/proj/include/
aura``): ``Convolver``, ``Auralizer``, ``EngineConfig``, ``ErrorCode``,
``Error``, ``make_config``, ``partition_count``, ``latency_budget``,
``list_backends``, ``make_backend`` -- same names, argument meaning and
error behaviour, backed by ``libaura_b200.so`` (hand-written sm_100a CUDA,
``csrc/``) through its C-ABI (``include/aura_b200.h``).

There is no CPU fallback: importing works anywhere, but constructing an
engine without the built library or without a B200 raises
``Error(ErrorCode.backend_unavailable)``.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "ErrorCode", "Error", "EngineConfig", "ChannelMode", "make_config",
    "validate_config", "partition_count", "latency_budget", "BackendKind",
    "BackendDescriptor", "list_backends", "make_backend", "Convolver",
    "Auralizer", "AfcParams", "lib", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AURA_B200_LIB") or os.path.join(HERE, "libaura_b200.so")  # override: A/B experiments only


class ErrorCode(enum.IntEnum):
    """engine.hpp:15-37, plus the GPU codes appended by include/aura_b200.h."""
    non_power_of_two_block = 0
    fft_size_mismatch = 1
    bad_channel_combination = 2
    zero_sample_rate = 3
    zero_length = 4
    length_mismatch = 5
    non_real_edge_bins = 6
    filter_length_mismatch = 7
    empty_filter = 8
    mode_channel_mismatch = 9
    channel_count_mismatch = 10
    shape_mismatch = 11
    non_finite_input = 12
    empty_input = 13
    unsupported_format = 14
    corrupt_header = 15
    sample_rate_mismatch = 16
    backend_unavailable = 17
    out_of_memory = 18
    io_error = 19
    invalid_argument = 20
    cuda_error = 21
    timeout = 22


class Error(RuntimeError):
    """aura::Error (engine.hpp:39-47): carries an ErrorCode."""

    def __init__(self, code: ErrorCode, what: str):
        super().__init__(what)
        self.code = ErrorCode(code)


def _raise(code, what):
    raise Error(code, what)


class ChannelMode(enum.IntEnum):
    """engine.hpp:283, plus MIMO."""
    broadcast = 0
    elementwise = 1
    mimo = 2


@dataclass
class EngineConfig:
    """engine.hpp:64-72."""
    sample_rate_hz: int = 48000
    block_size: int = 128
    fft_size: int = 256
    input_channels: int = 1
    output_channels: int = 1

    def bins(self) -> int:
        return self.block_size + 1


def _pow2(v):
    return v > 0 and (v & (v - 1)) == 0


def validate_config(cfg: EngineConfig, mimo: bool = False) -> EngineConfig:
    """engine.hpp:74-94 (MIMO lifts only the C_in in {1, C_out} rule)."""
    if cfg.sample_rate_hz == 0:
        _raise(ErrorCode.zero_sample_rate, "sample rate must be positive")
    if not _pow2(cfg.block_size) or cfg.block_size < 16 or cfg.block_size > 8192:
        _raise(ErrorCode.non_power_of_two_block,
               f"block size must be a power of two in [16, 8192], got {cfg.block_size}")
    if cfg.fft_size != 2 * cfg.block_size:
        _raise(ErrorCode.fft_size_mismatch,
               f"fft size must be 2 * block size, got {cfg.fft_size} for block size {cfg.block_size}")
    if cfg.output_channels == 0 or cfg.input_channels == 0 or (
            not mimo and cfg.input_channels not in (1, cfg.output_channels)):
        _raise(ErrorCode.bad_channel_combination,
               "input channels must be 1 or equal to output channels")
    return cfg


def make_config(sample_rate_hz: int, block_size: int, input_channels: int,
                output_channels: int, mimo: bool = False) -> EngineConfig:
    """engine.hpp:96-108."""
    cfg = EngineConfig(sample_rate_hz, block_size, 2 * block_size,
                       input_channels, output_channels)
    return validate_config(cfg, mimo)


def partition_count(filter_length: int, block_size: int) -> int:
    """engine.hpp:112-117."""
    if filter_length == 0 or block_size == 0:
        _raise(ErrorCode.zero_length, "partition_count requires nonzero lengths")
    return (filter_length + block_size - 1) // block_size


def latency_budget(cfg: EngineConfig) -> float:
    """engine.hpp:120-124: n_x / f_s seconds."""
    validate_config(cfg, cfg.input_channels not in (1, cfg.output_channels))
    return cfg.block_size / cfg.sample_rate_hz


# ------------------------------------------------------------------ library

class _Cfg(C.Structure):
    _fields_ = [("sample_rate_hz", C.c_uint32), ("block_size", C.c_size_t),
                ("fft_size", C.c_size_t), ("inputs", C.c_size_t),
                ("outputs", C.c_size_t)]


class _Afc(C.Structure):
    _fields_ = [("mu", C.c_float), ("lambda_", C.c_float), ("delta", C.c_float),
                ("constrained", C.c_int)]


_lib = None
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def lib():
    """Load libaura_b200.so (built in-tree by __graft_entry__.build() /
    `make -C paper_2509_04390_b200`). Fails loudly when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        _raise(ErrorCode.backend_unavailable,
               f"{LIB_PATH} is not built; run `make -C paper_2509_04390_b200`")
    L = C.CDLL(LIB_PATH)
    vp, sz = C.c_void_p, C.c_size_t
    fpp = C.POINTER(C.c_void_p)
    L.aura_b200_abi_version.restype = C.c_int
    L.aura_b200_last_error.restype = C.c_char_p
    L.aura_b200_device_count.argtypes = [C.POINTER(C.c_int)]
    L.aura_b200_device_name.argtypes = [C.c_int, C.c_char_p, sz]
    L.aura_b200_convolver_create.argtypes = [C.POINTER(_Cfg), C.c_int, fpp, sz, sz,
                                             C.c_int, C.POINTER(vp)]
    L.aura_b200_auralizer_create.argtypes = [C.POINTER(_Cfg), fpp, sz, sz, fpp, sz, sz,
                                             C.c_float, C.POINTER(_Afc), C.c_int,
                                             C.POINTER(vp)]
    L.aura_b200_destroy.argtypes = [vp]
    L.aura_b200_process.argtypes = [vp, _f32p, _f32p]
    L.aura_b200_io_buffers.argtypes = [vp, C.POINTER(C.POINTER(C.c_float)), C.POINTER(C.POINTER(C.c_float))]
    L.aura_b200_process_io.argtypes = [vp]
    L.aura_b200_deadline_stats.argtypes = [vp, C.POINTER(C.c_uint64)] + [C.POINTER(C.c_double)] * 3
    L.aura_b200_reset.argtypes = [vp]
    L.aura_b200_feedback_estimate.argtypes = [vp, _f32p]
    L.aura_b200_set_input_gain.argtypes = [vp, C.c_float]
    L.aura_b200_set_launch_mode.argtypes = [vp, C.c_int]
    L.aura_b200_launch_mode.argtypes = [vp]
    L.aura_b200_seek_block.argtypes = [vp, C.c_uint64]
    L.aura_b200_time_host_breakdown.argtypes = [vp, vp, sz, sz, C.c_double, vp]
    L.aura_b200_input_gain.argtypes = [vp]
    L.aura_b200_input_gain.restype = C.c_float
    for name in ("blocks_processed",):
        getattr(L, "aura_b200_" + name).argtypes = [vp]
        getattr(L, "aura_b200_" + name).restype = C.c_uint64
    for name in ("partition_count", "fc_partition_count", "filter_length"):
        getattr(L, "aura_b200_" + name).argtypes = [vp]
        getattr(L, "aura_b200_" + name).restype = sz
    L.aura_b200_mode.argtypes = [vp]
    L.aura_b200_filter_spectrum.argtypes = [vp, sz, sz, _f32p]
    L.aura_b200_afc_coeffs.argtypes = [vp, _f32p]
    L.aura_b200_afc_load_coeffs.argtypes = [vp, _f32p, C.c_int]
    L.aura_b200_fdl_slot.argtypes = [vp, C.c_int, sz, sz, _f32p]
    L.aura_b200_time_device_blocks.argtypes = [vp, C.c_void_p, sz, sz, _f32p, _f32p]
    L.aura_b200_time_device_span.argtypes = [vp, C.c_void_p, sz, sz, C.POINTER(C.c_float)]
    L.aura_b200_synchronize.argtypes = [vp]
    L.aura_b200_time_host_blocks.argtypes = [vp, _f32p, sz, sz, C.c_double, _f32p]
    L.aura_b200_profile_phases.argtypes = [vp, sz, _f32p, C.POINTER(C.c_int)]
    L.aura_b200_phase_name.argtypes = [vp, C.c_int]
    L.aura_b200_phase_name.restype = C.c_char_p
    L.aura_b200_phase_bytes.argtypes = [vp, C.c_int]
    L.aura_b200_phase_bytes.restype = C.c_double
    L.aura_b200_describe.argtypes = [vp, C.c_char_p, sz]
    L.aura_b200_launches_per_block.argtypes = [vp]
    L.aura_b200_time_phase.argtypes = [vp, C.c_int, sz, C.POINTER(C.c_float)]
    L.aura_b200_trace_blocks.argtypes = [vp, sz, np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
    L.aura_b200_trace_host_blocks.argtypes = [vp, _f32p, sz, sz,
                                              np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
    L.aura_b200_trace_back.argtypes = [vp, sz, vp, C.POINTER(C.c_size_t), vp, C.POINTER(C.c_size_t)]
    _lib = L
    return L


def _check(rc):
    if rc:
        _raise(ErrorCode(rc - 1), lib().aura_b200_last_error().decode())


# ----------------------------------------------------------------- backends

class BackendKind(enum.IntEnum):
    """backend.hpp:16."""
    reference = 0
    parallel = 1
    accelerator = 2


@dataclass
class BackendDescriptor:
    """backend.hpp:18-23."""
    name: str
    kind: BackendKind
    available: bool
    detail: str
    device: int = 0


def list_backends():
    """backend.hpp:186-193: this build offers only the accelerator (one entry
    per B200); the reference's CPU backends live in the reference library."""
    out = []
    try:
        n = C.c_int(0)
        _check(lib().aura_b200_device_count(C.byref(n)))
        for d in range(n.value):
            buf = C.create_string_buffer(256)
            _check(lib().aura_b200_device_name(d, buf, 256))
            out.append(BackendDescriptor("accelerator", BackendKind.accelerator, True,
                                         buf.value.decode(), d))
    except Error:
        pass
    return out


def make_backend(name: str = "accelerator", device: int = 0) -> BackendDescriptor:
    """backend.hpp:197-207. "accelerator"/"gpu" select a B200; the CPU
    backends are not part of this build (no CPU fallback)."""
    if name in ("accelerator", "gpu"):
        for b in list_backends():
            if b.device == device:
                return b
        _raise(ErrorCode.backend_unavailable,
               "accelerator backend is not available: no compatible device")
    if name in ("reference", "parallel", "cpu"):
        _raise(ErrorCode.backend_unavailable,
               f"backend '{name}' is a CPU backend; this build runs only on the B200")
    _raise(ErrorCode.backend_unavailable,
           f"unknown backend '{name}' (expected accelerator)")


def _rows(filters) -> tuple:
    rows = [np.ascontiguousarray(f, dtype=np.float32).ravel() for f in filters]
    return rows


def _row_ptrs(rows):
    arr = (C.c_void_p * max(1, len(rows)))()
    for i, r in enumerate(rows):
        arr[i] = r.ctypes.data
    return arr


def _cfg(cfg: EngineConfig) -> _Cfg:
    return _Cfg(cfg.sample_rate_hz, cfg.block_size, cfg.fft_size,
                cfg.input_channels, cfg.output_channels)


class _Engine:
    _h = None

    def _fin(self):
        if self._h:
            lib().aura_b200_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self._fin()
        except Exception:
            pass

    def close(self):
        self._fin()

    @property
    def handle(self):
        return self._h

    def blocks_processed(self) -> int:
        return int(lib().aura_b200_blocks_processed(self._h))

    def partition_count(self) -> int:
        return int(lib().aura_b200_partition_count(self._h))

    def io_buffers(self):
        """Zero-copy I/O (aura_b200_io_buffers): numpy views of the engine's
        pinned, device-mapped input (C_in, N) and output (C_out, N) blocks.
        Write the input view, call process_io(), read the output view before
        the next call."""
        pi, po = C.POINTER(C.c_float)(), C.POINTER(C.c_float)()
        _check(lib().aura_b200_io_buffers(self._h, C.byref(pi), C.byref(po)))
        N = self.cfg.block_size
        return (np.ctypeslib.as_array(pi, shape=(self.cfg.input_channels, N)),
                np.ctypeslib.as_array(po, shape=(self.cfg.output_channels, N)))

    def process_io(self):
        """One block from / to the io_buffers() views (no host copies)."""
        _check(lib().aura_b200_process_io(self._h))

    def deadline_stats(self) -> dict:
        """Failure detection: process()/process_io() calls over the real-time
        budget N / f_s since creation or reset, max / last latency (us)."""
        m = C.c_uint64()
        mx, last, bud = C.c_double(), C.c_double(), C.c_double()
        _check(lib().aura_b200_deadline_stats(self._h, C.byref(m), C.byref(mx), C.byref(last), C.byref(bud)))
        return {"misses": int(m.value), "max_us": mx.value, "last_us": last.value, "budget_us": bud.value}

    def reset(self):
        _check(lib().aura_b200_reset(self._h))

    def fdl_slot(self, which: int, channel: int, age: int) -> np.ndarray:
        """FrequencyDelayLine::slot(channel, age) (engine.hpp:261-266) of the
        input FDL (which = 0) or the canceller FDL (which = 1): N+1 complex64."""
        n = self.cfg.block_size
        out = np.zeros(2 * (n + 1), np.float32)
        _check(lib().aura_b200_fdl_slot(self._h, which, channel, age, out))
        return out.view(np.complex64)

    TRACE_KERNELS = ("k_front", "k_back_head", "k_back", "k_reduce", "afc_done", "k_afc_finish",
                     "output", "afc_summed", "afc_c2r", "front_x", "afc_wait", "k_afc_constrain")
    _TRACE_SLOTS = 13  # kTraceKernels: the last slot is the next block's front start

    def trace_blocks(self, blocks: int = 32, host_inputs: Optional[np.ndarray] = None):
        """Per-kernel [start, end] (us from the block's front start) of
        back-to-back blocks, from %globaltimer stamps inside the kernels."""
        blocks = min(blocks, 64)
        out = np.zeros(blocks * self._TRACE_SLOTS * 2, np.float64)
        if host_inputs is None:
            _check(lib().aura_b200_trace_blocks(self._h, blocks, out))
        else:  # through process()'s mapped-memory handshake
            x = np.ascontiguousarray(host_inputs, np.float32)
            _check(lib().aura_b200_trace_host_blocks(self._h, x, x.shape[0], blocks, out))
        out = out.reshape(blocks, self._TRACE_SLOTS, 2)
        res = {name: out[:, k, :] for k, name in enumerate(self.TRACE_KERNELS)
               if np.all(out[:, k, 0] >= 0)}
        if blocks > 1:  # front start -> next block's front start (back to back)
            res["cycle"] = out[:-1, self._TRACE_SLOTS - 1, :]
        return res

    def trace_back(self, blocks: int = 8):
        """Diagnostics: k_back's per-segment end times and per-CTA {start,
        first data, exit} (us from the block's front start), last block."""
        ns, nc = C.c_size_t(0), C.c_size_t(0)
        _check(lib().aura_b200_trace_back(self._h, blocks, None, C.byref(ns), None, C.byref(nc)))
        segs = np.zeros((ns.value, 8), np.float64)
        ctas = np.zeros((nc.value, 3), np.float64)
        _check(lib().aura_b200_trace_back(self._h, blocks, segs.ctypes.data, C.byref(ns),
                                          ctas.ctypes.data, C.byref(nc)))
        return segs, ctas

    def set_launch_mode(self, mode: int):
        """0: one CUDA graph per block (default); 1: the same kernels
        launched on the stream (bit-identical)."""
        _check(lib().aura_b200_set_launch_mode(self._h, mode))

    def launch_mode(self) -> int:
        return int(lib().aura_b200_launch_mode(self._h))

    def seek_block(self, n: int):
        """Testing: number the device blocks from n (fresh or reset engine)."""
        _check(lib().aura_b200_seek_block(self._h, n))

    HOST_PHASES = ("staged", "launched", "event", "output_seen", "copied")

    def time_host_breakdown(self, inputs: np.ndarray, blocks: int, pace_us: float = 0.0):
        """Diagnostics: steady_clock offsets (us) inside process(), graph mode."""
        inputs = np.ascontiguousarray(inputs, np.float32)
        out = np.zeros((blocks, 5), np.float64)
        _check(lib().aura_b200_time_host_breakdown(self._h, inputs.ctypes.data, inputs.shape[0], blocks,
                                                   pace_us, out.ctypes.data))
        return {k: out[:, i] for i, k in enumerate(self.HOST_PHASES)}

    PHASES = {"k_front": 0, "k_back": 2, "k_reduce": 3}

    def time_phase(self, name: str, reps: int = 20) -> float:
        """Mean device time (us) of back-to-back launches of one phase
        kernel, CUDA events on the engine stream; the engine's state (block
        counter, power, canceller W and partials) is restored afterwards."""
        v = C.c_float(0)
        _check(lib().aura_b200_time_phase(self._h, self.PHASES[name], reps, C.byref(v)))
        return float(v.value)

    def launches_per_block(self) -> int:
        return int(lib().aura_b200_launches_per_block(self._h))

    def describe(self) -> str:
        buf = C.create_string_buffer(1024)
        _check(lib().aura_b200_describe(self._h, buf, 1024))
        return buf.value.decode()

    # ---- measurement hooks used by bench.py
    def synchronize(self):
        """Wait for every processed block's background work (next-block
        precompute, canceller update)."""
        _check(lib().aura_b200_synchronize(self._h))

    def time_device_span(self, blocks: int, inputs: Optional[np.ndarray] = None) -> float:
        """Mean device time per block (us) of `blocks` back-to-back blocks
        timed with one event pair around all of them."""
        v = C.c_float(0)
        ptr, n = None, 0
        if inputs is not None:
            inputs = np.ascontiguousarray(inputs, np.float32)
            ptr, n = inputs.ctypes.data, inputs.shape[0]
        _check(lib().aura_b200_time_device_span(self._h, ptr, n, blocks, C.byref(v)))
        return float(v.value) / blocks

    def time_device_blocks(self, blocks: int, inputs: Optional[np.ndarray] = None):
        """Back-to-back device-resident blocks timed with CUDA events.
        Returns (latency_us, block_us): block start -> output written, and
        all of the block's work (front + background)."""
        lat = np.zeros(blocks, np.float32)
        out = np.zeros(blocks, np.float32)
        if inputs is not None:
            inputs = np.ascontiguousarray(inputs, np.float32)
            n_in = inputs.shape[0]
            _check(lib().aura_b200_time_device_blocks(self._h, inputs.ctypes.data, n_in,
                                                      blocks, lat, out))
        else:
            _check(lib().aura_b200_time_device_blocks(self._h, None, 0, blocks, lat, out))
        return lat, out

    def time_host_blocks(self, inputs: np.ndarray, blocks: int, pace_us: float = 0.0):
        """Per-call latency of process() with host buffers (C-side timing)."""
        inputs = np.ascontiguousarray(inputs, np.float32)
        out = np.zeros(blocks, np.float32)
        _check(lib().aura_b200_time_host_blocks(self._h, inputs, inputs.shape[0], blocks,
                                                pace_us, out))
        return out

    def profile_phases(self, blocks: int):
        us = np.zeros(16, np.float32)
        n = C.c_int(0)
        _check(lib().aura_b200_profile_phases(self._h, blocks, us, C.byref(n)))
        return {lib().aura_b200_phase_name(self._h, i).decode():
                (float(us[i]), float(lib().aura_b200_phase_bytes(self._h, i)))
                for i in range(n.value)}


class Convolver(_Engine):
    """aura::Convolver (convolver.hpp:65-220) on the B200.

    filters: C_out (broadcast/elementwise) or Q*C_out (mimo, row q*L+l)
    time-domain filters of one common length."""

    def __init__(self, filters: Sequence, cfg: EngineConfig,
                 mode: ChannelMode = ChannelMode.broadcast,
                 backend: Optional[BackendDescriptor] = None):
        validate_config(cfg, mode == ChannelMode.mimo)
        rows = _rows(filters)
        if len(rows) == 0:
            _raise(ErrorCode.empty_filter, "need at least one filter")
        n_h = rows[0].size
        if n_h == 0:
            _raise(ErrorCode.empty_filter, "filters must have at least one tap")
        if any(r.size != n_h for r in rows):
            _raise(ErrorCode.filter_length_mismatch, "all filters must share one length")
        device = backend.device if backend is not None else 0
        h = C.c_void_p()
        _check(lib().aura_b200_convolver_create(C.byref(_cfg(cfg)), int(mode), _row_ptrs(rows),
                                                len(rows), n_h, device, C.byref(h)))
        self._h = h
        self.cfg = cfg
        self.mode = ChannelMode(mode)
        self._n_h = n_h
        self._out = np.zeros((cfg.output_channels, cfg.block_size), np.float32)

    def config(self) -> EngineConfig:
        return self.cfg

    def filter_length(self) -> int:
        return self._n_h

    def process(self, block: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """convolver.hpp:111-123: (C_in, N) -> (C_out, N)."""
        x = np.ascontiguousarray(block, dtype=np.float32)
        if x.ndim != 2 or x.shape != (self.cfg.input_channels, self.cfg.block_size):
            _raise(ErrorCode.shape_mismatch, "input block must be input_channels x block_size")
        if out is None:
            out = np.empty((self.cfg.output_channels, self.cfg.block_size), np.float32)
        elif out.shape != (self.cfg.output_channels, self.cfg.block_size) or \
                out.dtype != np.float32 or not out.flags.c_contiguous:
            _raise(ErrorCode.shape_mismatch, "output block must be output_channels x block_size")
        _check(lib().aura_b200_process(self._h, x, out))
        return out

    convolve = process

    def spectrum(self, row: int, k: int) -> np.ndarray:
        """filters().spectrum(row, k) (engine.hpp:210-219): N+1 complex64."""
        out = np.zeros(2 * (self.cfg.block_size + 1), np.float32)
        _check(lib().aura_b200_filter_spectrum(self._h, row, k, out))
        return out.view(np.complex64)


@dataclass
class AfcParams:
    """Feedback-canceller adaptation; mu = 0 is the
    reference's fixed canceller. delta None -> 1e-6 * N.
    constrained: the constrained gradient of Appendix A step 2 (each
    partition's update keeps only its first N taps)."""
    mu: float = 0.0
    lam: float = 0.9
    delta: Optional[float] = None
    constrained: bool = False


def default_delta(block_size: int) -> float:
    """NLMS regulariser default: SURVEY Appendix A's delta = 1e-6 * N
    (DESIGN.md section 4 has the W-error evidence at this value)."""
    return 1e-6 * block_size


class Auralizer(_Engine):
    """aura::Auralizer (auralizer.hpp:25-123) on the B200, with the optional
    NLMS adaptation of the canceller and Q > 1 MIMO.

    synth: Q*L rows (row q*L + l); fc: Q*L rows (row p*L + l)."""

    def __init__(self, synth_filters: Sequence, fc_filters: Sequence, cfg: EngineConfig,
                 backend: Optional[BackendDescriptor] = None, input_gain: float = 1.0,
                 afc: Optional[AfcParams] = None):
        validate_config(cfg, True)
        srows, frows = _rows(synth_filters), _rows(fc_filters)
        if len(srows) != len(frows):
            _raise(ErrorCode.channel_count_mismatch,
                   "synthesis and feedback-cancellation filter sets must have the same channel count")
        for rows in (srows, frows):
            if len(rows) == 0:
                _raise(ErrorCode.empty_filter, "need at least one filter")
            if rows[0].size == 0:
                _raise(ErrorCode.empty_filter, "filters must have at least one tap")
            if any(r.size != rows[0].size for r in rows):
                _raise(ErrorCode.filter_length_mismatch, "all filters must share one length")
        device = backend.device if backend is not None else 0
        a = afc or AfcParams()
        delta = a.delta if a.delta is not None else default_delta(cfg.block_size)
        pa = _Afc(a.mu, a.lam, delta, 1 if a.constrained else 0)
        h = C.c_void_p()
        _check(lib().aura_b200_auralizer_create(
            C.byref(_cfg(cfg)), _row_ptrs(srows), len(srows), srows[0].size,
            _row_ptrs(frows), len(frows), frows[0].size, input_gain, C.byref(pa),
            device, C.byref(h)))
        self._h = h
        self.cfg = cfg
        self.afc = a
        self._kf = int(lib().aura_b200_fc_partition_count(h))

    def config(self) -> EngineConfig:
        return self.cfg

    def synth_partitions(self) -> int:
        return self.partition_count()

    def fc_partitions(self) -> int:
        return self._kf

    def input_gain(self) -> float:
        return float(lib().aura_b200_input_gain(self._h))

    def set_input_gain(self, g: float):
        _check(lib().aura_b200_set_input_gain(self._h, g))

    def feedback_estimate(self) -> np.ndarray:
        """auralizer.hpp:56-58: (Q, N) -- the estimate for the next block."""
        out = np.zeros((self.cfg.input_channels, self.cfg.block_size), np.float32)
        _check(lib().aura_b200_feedback_estimate(self._h, out))
        return out

    def process(self, mic: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """auralizer.hpp:61-87: mic (Q, N) -> speakers (L, N)."""
        x = np.ascontiguousarray(mic, dtype=np.float32)
        if x.ndim != 2 or x.shape != (self.cfg.input_channels, self.cfg.block_size):
            _raise(ErrorCode.shape_mismatch, "microphone block must be inputs x block_size")
        if out is None:
            out = np.empty((self.cfg.output_channels, self.cfg.block_size), np.float32)
        elif out.shape != (self.cfg.output_channels, self.cfg.block_size) or \
                out.dtype != np.float32 or not out.flags.c_contiguous:
            _raise(ErrorCode.shape_mismatch, "speaker block must be output_channels x block_size")
        _check(lib().aura_b200_process(self._h, x, out))
        return out

    auralize = process

    def coeffs(self) -> np.ndarray:
        """Canceller spectra W (P, L, K_f, N+1) complex64."""
        P, L, N = self.cfg.input_channels, self.cfg.output_channels, self.cfg.block_size
        out = np.zeros(P * L * self._kf * (N + 1) * 2, np.float32)
        _check(lib().aura_b200_afc_coeffs(self._h, out))
        return out.view(np.complex64).reshape(P, L, self._kf, N + 1)

    def load_coeffs(self, W: np.ndarray, as_initial: bool = False):
        """Load canceller spectra W (P, L, K_f, N+1) complex64: checkpoint /
        warm start; as_initial makes reset() return to them."""
        P, L, N = self.cfg.input_channels, self.cfg.output_channels, self.cfg.block_size
        w = np.ascontiguousarray(W, np.complex64)
        if w.shape != (P, L, self._kf, N + 1):
            _raise(ErrorCode.shape_mismatch, f"canceller spectra must be {(P, L, self._kf, N + 1)}")
        _check(lib().aura_b200_afc_load_coeffs(self._h, w.view(np.float32).ravel(), 1 if as_initial else 0))
