"""Loudspeaker-channel sharding of the block loop across GPUs.

One process per GPU. Each rank owns a contiguous slice [l0, l1) of the L
loudspeakers: its rows of the synthesis filters H and canceller filters F^,
its canceller delay line, and a replica of the (tiny) input delay line. Every
rank receives the same microphone block and writes its own loudspeaker slice.

Synthesis needs no exchange. With the feedback canceller on, f^ and the NLMS
power sum over ALL loudspeakers, so the engines exchange P*N + 2N floats per
block inside their CUDA graph (k_afc_finish: P2P stores over NVLink plus
system-scope flags, summed in rank order -- bit-identical on every rank).
``torch.distributed`` is only the plumbing that all-gathers the 64-byte CUDA
IPC handles of the exchange buffers once at setup.

``VirtualShards`` runs G shards on ONE device in one process with the same
kernels and protocol (the build box has one GPU).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import (AfcParams, Auralizer, ChannelMode, Convolver, EngineConfig, Error, ErrorCode,
               _check, lib, make_backend, make_config)

HANDLE_BYTES = 64
NCCL_ID_BYTES = 128
MAX_SHARDS = 8
TRANSPORTS = ("p2p", "nccl")


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 creates it, the host distributes it)."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _check(_lib_shard().aura_b200_nccl_unique_id(buf))
    return buf.raw


def connect_nccl(engine, world: int, rank: int, uid: bytes):
    if len(uid) != NCCL_ID_BYTES:
        raise Error(ErrorCode.invalid_argument, "NCCL unique id must be 128 bytes")
    _check(_lib_shard().aura_b200_shard_connect_nccl(engine.handle, world, rank, uid))


def shard_range(L: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous near-even split of L loudspeakers: the first L % world
    ranks get one extra channel."""
    if world < 1 or not 0 <= rank < world:
        raise Error(ErrorCode.invalid_argument, "bad shard rank/world")
    if L < world:
        raise Error(ErrorCode.invalid_argument, f"{L} loudspeakers cannot be split over {world} shards")
    base, extra = divmod(L, world)
    l0 = rank * base + min(rank, extra)
    return l0, l0 + base + (1 if rank < extra else 0)


def shard_rows(rows: Sequence, Q: int, L: int, l0: int, l1: int) -> list:
    """Rows q*L + l (l in [l0, l1)) of a Q x L row set, re-indexed q*(l1-l0) + l."""
    if len(rows) != Q * L:
        raise Error(ErrorCode.mode_channel_mismatch, "filter count must equal inputs x outputs")
    return [rows[q * L + l] for q in range(Q) for l in range(l0, l1)]


def _lib_shard():
    L = lib()
    if not hasattr(L, "_shard_bound"):
        vp = C.c_void_p
        L.aura_b200_shard_export.argtypes = [vp, C.c_int, C.c_int, C.c_char_p]
        L.aura_b200_shard_connect.argtypes = [vp, C.c_char_p]
        L.aura_b200_shard_connect_local.argtypes = [C.POINTER(vp), C.c_int]
        L.aura_b200_shard_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.aura_b200_nccl_unique_id.argtypes = [C.c_char_p]
        L.aura_b200_shard_connect_nccl.argtypes = [vp, C.c_int, C.c_int, C.c_char_p]
        L._shard_bound = True
    return L


def exchange_handles(handle: bytes, group=None) -> bytes:
    """All-gather one 64-byte handle per rank, concatenated in rank order."""
    import torch.distributed as dist
    if len(handle) != HANDLE_BYTES:
        raise Error(ErrorCode.invalid_argument, "shard handle must be 64 bytes")
    out: List[Optional[bytes]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return b"".join(out)


class ShardedAuralizer:
    """``Auralizer`` whose loudspeakers are split over the ranks of a
    torch.distributed group (one process per GPU). Each rank passes the FULL
    filter sets (or any object indexable by row) and gets back its own
    loudspeaker slice from ``process``. All ranks must call ``process`` with
    the same microphone blocks, and ``reset`` together. ``transport``: "p2p"
    (our in-graph exchange kernel, the default) or "nccl" (ncclAllReduce
    captured in the graph; the ablation)."""

    def __init__(self, synth_filters: Sequence, fc_filters: Sequence, cfg: EngineConfig,
                 device: int = 0, input_gain: float = 1.0, afc: Optional[AfcParams] = None,
                 group=None, transport: str = "p2p"):
        import torch.distributed as dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.group = group
        Q, L = cfg.input_channels, cfg.output_channels
        self.l0, self.l1 = shard_range(L, self.world, self.rank)
        local = make_config(cfg.sample_rate_hz, cfg.block_size, Q, self.l1 - self.l0, mimo=Q > 1)
        self.cfg = cfg
        err = None
        try:
            self.engine = Auralizer(shard_rows(synth_filters, Q, L, self.l0, self.l1),
                                    shard_rows(fc_filters, Q, L, self.l0, self.l1), local,
                                    make_backend("gpu", device), input_gain, afc)
        except Error as e:  # tell the other ranks before raising
            err = e
        errs = [None] * self.world
        dist.all_gather_object(errs, None if err is None else (int(err.code), str(err)), group=group)
        bad = [e for e in errs if e is not None]
        if bad:
            raise err if err is not None else Error(ErrorCode(bad[0][0]), "peer shard: " + bad[0][1])
        if transport not in TRANSPORTS:
            raise Error(ErrorCode.invalid_argument, f"transport must be one of {TRANSPORTS}")
        self.transport = transport
        if transport == "nccl":
            box = [nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(box, src=0, group=group)
            connect_nccl(self.engine, self.world, self.rank, box[0])
            dist.barrier(group=group)
        elif self.world > 1:
            h = C.create_string_buffer(HANDLE_BYTES)
            _check(_lib_shard().aura_b200_shard_export(self.engine.handle, self.world, self.rank, h))
            allh = exchange_handles(h.raw, group)
            _check(_lib_shard().aura_b200_shard_connect(self.engine.handle, allh))
            dist.barrier(group=group)

    @property
    def channels(self) -> Tuple[int, int]:
        return self.l0, self.l1

    def process(self, mic: np.ndarray) -> np.ndarray:
        return self.engine.process(mic)

    def feedback_estimate(self) -> np.ndarray:
        return self.engine.feedback_estimate()

    def coeffs(self) -> np.ndarray:
        return self.engine.coeffs()

    def reset(self):
        import torch.distributed as dist
        self.engine.synchronize()
        dist.barrier(group=self.group)
        self.engine.reset()
        dist.barrier(group=self.group)

    def close(self):
        self.engine.close()


class ShardedConvolver:
    """``Convolver`` (broadcast or MIMO) split by loudspeaker: the shards are
    independent -- no exchange at all."""

    def __init__(self, filters: Sequence, cfg: EngineConfig, world: int, rank: int,
                 mode: ChannelMode = ChannelMode.broadcast, device: int = 0):
        Q = cfg.input_channels if mode == ChannelMode.mimo else 1
        L = cfg.output_channels
        if mode == ChannelMode.elementwise:
            raise Error(ErrorCode.invalid_argument, "shard elementwise convolvers by creating "
                                                    "one convolver per channel range")
        self.l0, self.l1 = shard_range(L, world, rank)
        local = make_config(cfg.sample_rate_hz, cfg.block_size, cfg.input_channels,
                            self.l1 - self.l0, mimo=mode == ChannelMode.mimo)
        self.engine = Convolver(shard_rows(filters, Q, L, self.l0, self.l1), local, mode,
                                make_backend("gpu", device))

    def process(self, block: np.ndarray) -> np.ndarray:
        return self.engine.process(block)

    def close(self):
        self.engine.close()


class VirtualShards:
    """G shards of one auralizer on one device, in one process: the same
    kernels and exchange protocol as ShardedAuralizer, wired through
    aura_b200_shard_connect_local. ``process`` runs every shard on the block
    and returns the concatenated loudspeaker signals (L x N)."""

    def __init__(self, synth_filters: Sequence, fc_filters: Sequence, cfg: EngineConfig,
                 world: int, device: int = 0, input_gain: float = 1.0,
                 afc: Optional[AfcParams] = None, devices: Optional[Sequence[int]] = None):
        Q, L = cfg.input_channels, cfg.output_channels
        self.world = world
        self.ranges = [shard_range(L, world, g) for g in range(world)]
        self.shards = []
        for g, (l0, l1) in enumerate(self.ranges):
            dev = devices[g] if devices else device
            local = make_config(cfg.sample_rate_hz, cfg.block_size, Q, l1 - l0, mimo=Q > 1)
            self.shards.append(Auralizer(shard_rows(synth_filters, Q, L, l0, l1),
                                         shard_rows(fc_filters, Q, L, l0, l1), local,
                                         make_backend("gpu", dev), input_gain, afc))
        arr = (C.c_void_p * world)(*[s.handle.value for s in self.shards])
        _check(_lib_shard().aura_b200_shard_connect_local(arr, world))
        self.cfg = cfg

    def process(self, mic: np.ndarray) -> np.ndarray:
        return np.concatenate([s.process(mic) for s in self.shards], axis=0)

    def feedback_estimates(self) -> list:
        return [s.feedback_estimate() for s in self.shards]

    def feedback_estimate(self) -> np.ndarray:
        return self.shards[0].feedback_estimate()

    def coeffs(self) -> np.ndarray:
        return np.concatenate([s.coeffs() for s in self.shards], axis=1)

    def reset(self):
        for s in self.shards:
            s.synchronize()
        for s in self.shards:
            s.reset()

    def close(self):
        for s in self.shards:
            s.close()
