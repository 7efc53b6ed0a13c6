"""CPU: host-side logic of loudspeaker sharding -- the channel
plan, row slicing (incl. MIMO row order), and the handle exchange over a
world_size-2 gloo group; without a B200 every rank fails loudly (no CPU
fallback, no hang)."""
import os
import socket

import numpy as np
import pytest

import paper_2509_04390_b200 as A
from paper_2509_04390_b200 import shard as S


@pytest.mark.parametrize("L,world", [(64, 1), (64, 2), (64, 8), (10, 3), (512, 8), (7, 7)])
def test_shard_range_partitions_all_channels(L, world):
    seen = []
    for r in range(world):
        l0, l1 = S.shard_range(L, world, r)
        assert l1 > l0
        seen.extend(range(l0, l1))
    assert seen == list(range(L))
    sizes = [S.shard_range(L, world, r)[1] - S.shard_range(L, world, r)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_splits():
    with pytest.raises(A.Error):
        S.shard_range(3, 4, 0)
    with pytest.raises(A.Error):
        S.shard_range(8, 2, 2)


def test_shard_rows_mimo_order():
    Q, L = 3, 5
    rows = [f"q{q}l{l}" for q in range(Q) for l in range(L)]
    got = S.shard_rows(rows, Q, L, 1, 3)
    assert got == ["q0l1", "q0l2", "q1l1", "q1l2", "q2l1", "q2l2"]
    with pytest.raises(A.Error):
        S.shard_rows(rows[:-1], Q, L, 0, 1)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes([rank]) * S.HANDLE_BYTES
        allh = S.exchange_handles(mine)
        ok_order = allh == b"".join(bytes([r]) * S.HANDLE_BYTES for r in range(world))
        err = None
        try:
            rng = np.random.default_rng(0)
            synth = list(rng.standard_normal((8, 256)).astype(np.float32))
            fc = list(rng.standard_normal((8, 64)).astype(np.float32))
            S.ShardedAuralizer(synth, fc, A.make_config(48000, 64, 1, 8), device=0,
                               afc=A.AfcParams(0.01))
        except A.Error as e:
            err = int(e.code)
        q.put((rank, ok_order, err))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_handle_exchange_and_loud_failure():
    import torch
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=30)
    assert [r[1] for r in res] == [True, True]
    if not torch.cuda.is_available():
        # both ranks raise backend_unavailable together (nobody hangs in a collective)
        assert [r[2] for r in res] == [int(A.ErrorCode.backend_unavailable)] * 2
