"""GPU: loudspeaker-channel sharding against the unsharded
C oracle. The build box has one B200, so shards run (a) as virtual shards in
one process (same kernels + exchange protocol, same-device stores) and (b) as
two processes on the same GPU wired through CUDA IPC -- the exact multi-GPU
code path minus NVLink."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_2509_04390_b200 as A
from paper_2509_04390_b200 import shard as S
from conftest import decaying_filters, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-5


def workload(Q, L, N, seed):
    rng = np.random.default_rng(seed)
    synth = decaying_filters(rng, Q * L, 12 * N + 5, scale=0.5)
    fc = decaying_filters(rng, Q * L, 4 * N + 1, scale=0.1)
    mic = rng.standard_normal((120, Q, N)).astype(np.float32)
    return synth, fc, mic


@pytest.mark.parametrize("Q,L,N,G,mu", [(1, 8, 64, 2, 0.01), (1, 16, 32, 4, 0.05),
                                        (2, 6, 64, 3, 0.02), (4, 8, 32, 2, 0.01),
                                        (1, 10, 128, 8, 0.0)])
def test_virtual_shards_match_unsharded_oracle(Q, L, N, G, mu):
    synth, fc, mic = workload(Q, L, N, 100 * G + L)
    kw = dict(gain=0.9, mu=mu, lam=0.9, delta=1e-2)
    cfg = A.make_config(48000, N, Q, L, mimo=Q > 1)
    v = S.VirtualShards(list(synth), list(fc), cfg, G, input_gain=kw["gain"],
                        afc=A.AfcParams(mu, kw["lam"], kw["delta"]))
    o = O.OracleAuralizer(synth, fc, N, Q, L, **kw)
    ys, yo, fv, fo = [], [], [], []
    for b in range(mic.shape[0]):
        ys.append(v.process(mic[b]))
        yo.append(o.process(mic[b]))
        ests = v.feedback_estimates()
        for e in ests[1:]:  # every shard holds the same f^, bit for bit
            assert np.array_equal(e, ests[0])
        fv.append(ests[0])
        fo.append(o.feedback_estimate())
    assert rel_err(np.stack(ys), np.stack(yo)) <= TOL
    assert rel_err(np.stack(fv), np.stack(fo)) <= TOL
    assert rel_err(v.coeffs(), o.coeffs()) <= TOL
    v.close()


def test_virtual_shards_reset_is_exact():
    synth, fc, mic = workload(1, 8, 64, 5)
    cfg = A.make_config(48000, 64, 1, 8)
    v = S.VirtualShards(list(synth), list(fc), cfg, 2, afc=A.AfcParams(0.02, 0.9, 1e-2))
    a = np.stack([v.process(mic[b]) for b in range(30)])
    v.reset()
    b = np.stack([v.process(mic[i]) for i in range(30)])
    assert np.array_equal(a, b)
    v.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q, devices=(0, 0), transport="p2p"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Q, L, N = 1, 12, 64
        synth, fc, mic = workload(Q, L, N, 77)
        cfg = A.make_config(48000, N, Q, L)
        sh = S.ShardedAuralizer(list(synth), list(fc), cfg, device=devices[rank], input_gain=0.9,
                                afc=A.AfcParams(0.02, 0.9, 1e-2), transport=transport)
        ys, fs = [], []
        for b in range(mic.shape[0]):
            ys.append(sh.process(mic[b]))
            fs.append(sh.feedback_estimate())
        q.put((rank, sh.channels, np.stack(ys), np.stack(fs), sh.coeffs()))
        sh.close()
    except Exception as e:  # surface in the parent
        q.put((rank, "error", repr(e), None, None))
    finally:
        dist.destroy_process_group()


def _device_count():
    import torch
    return torch.cuda.device_count()


def test_two_processes_ipc_on_one_gpu():
    """One process per shard, exchange buffers opened through CUDA IPC
    (the multi-GPU wiring), both on cuda:0."""
    _two_process_run((0, 0), "p2p")


@pytest.mark.skipif(_device_count() < 2, reason="needs two GPUs (NVLink peers)")
@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_two_gpus_cross_device_exchange(transport):
    """Shards on cuda:0 and cuda:1, one process each: the canceller exchange
    crosses NVLink (P2P stores into the peer's IPC-mapped buffer, or the
    NCCL all-reduce); f^ bit-identical on both ranks, outputs within 1e-5
    of the unsharded oracle."""
    _two_process_run((0, 1), transport)


def _two_process_run(devices, transport):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q, devices, transport)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r in res.values():
        assert r[1] != "error", r[2]
    Q, L, N = 1, 12, 64
    synth, fc, mic = workload(Q, L, N, 77)
    o = O.OracleAuralizer(synth, fc, N, Q, L, gain=0.9, mu=0.02, lam=0.9, delta=1e-2)
    yo, fo = [], []
    for b in range(mic.shape[0]):
        yo.append(o.process(mic[b]))
        fo.append(o.feedback_estimate())
    yo, fo = np.stack(yo), np.stack(fo)
    (a0, a1), (b0, b1) = res[0][1], res[1][1]
    assert (a0, a1, b0, b1) == (0, 6, 6, 12)
    y = np.concatenate([res[0][2], res[1][2]], axis=1)
    assert rel_err(y, yo) <= TOL
    assert np.array_equal(res[0][3], res[1][3])
    assert rel_err(res[0][3], fo) <= TOL
    W = np.concatenate([res[0][4], res[1][4]], axis=1)
    assert rel_err(W, o.coeffs()) <= TOL


def test_sharded_convolver_is_independent_slices():
    rng = np.random.default_rng(3)
    N, L = 64, 10
    f = decaying_filters(rng, L, 20 * N)
    cfg = A.make_config(48000, N, 1, L)
    x = rng.standard_normal((40, 1, N)).astype(np.float32)
    o = O.OracleConvolver(f, N, 1, L, O.BROADCAST)
    parts = [S.ShardedConvolver(list(f), cfg, 3, r) for r in range(3)]
    for b in range(40):
        y = np.concatenate([p.process(x[b]) for p in parts], axis=0)
        assert rel_err(y, o.process(x[b])) <= TOL


def test_nccl_exchange_world_one_is_bit_identical():
    """The NCCL transport with one rank (a local all-reduce captured in the
    block graph, then k_afc_apply): bit-identical to the unsharded engine --
    the same partial c2r, sum and power smoothing operations."""
    synth, fc, mic = workload(1, 8, 64, 21)
    cfg = A.make_config(48000, 64, 1, 8)
    afc = A.AfcParams(0.02, 0.9, 1e-2)
    plain = A.Auralizer(list(synth), list(fc), cfg, input_gain=0.9, afc=afc)
    nc = A.Auralizer(list(synth), list(fc), cfg, input_gain=0.9, afc=afc)
    S.connect_nccl(nc, 1, 0, S.nccl_unique_id())
    for b in range(40):
        assert np.array_equal(nc.process(mic[b]), plain.process(mic[b])), b
        assert np.array_equal(nc.feedback_estimate(), plain.feedback_estimate()), b
    assert np.array_equal(nc.coeffs(), plain.coeffs())
    nc.reset()
    plain.reset()
    for b in range(5):
        assert np.array_equal(nc.process(mic[b]), plain.process(mic[b]))
    nc.close()
    plain.close()
