"""Multi-process reducer semantics on CPU (gloo, world_size 2): the Reducer
duck type (comm.py:66-114) with canonical rank-order sums (comm.py:41-46),
handshake, broadcast, and collective errors — the host logic the NCCL path
shares."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1803_06333_b200.comm import NcclReducer, ProtocolError, canonical_sum
    from paper_1803_06333_b200.data import partition_bounds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        det = NcclReducer(deterministic=True)
        fast = NcclReducer(deterministic=False)
        out["hs"] = det.handshake()
        vecs = [np.random.default_rng(10 + r).standard_normal(1000) * 1e3 for r in range(world)]
        out["det"] = det.allreduce_sum(vecs[rank])
        out["fast"] = fast.allreduce_sum(vecs[rank])
        out["canon"] = canonical_sum(vecs)
        out["bcast"] = det.broadcast(np.full(3, float(rank + 7)))
        t = torch.full((4,), float(rank + 1), dtype=torch.float64)
        fast.allreduce_inplace(t)
        out["inplace"] = t.numpy().copy()
        try:
            det.allreduce_sum(np.zeros(5 + rank))
            out["mismatch"] = "no error"
        except ProtocolError as exc:
            out["mismatch"] = str(exc)
        # each rank's node partition (engine.py:187-210 with node_index=rank)
        b = partition_bounds(1_000_000, world, 1)
        out["part"] = (int(b[rank]), int(b[rank + 1]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_reducer_semantics():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        o = res[r]
        assert o["hs"] == {"rank": r, "world": world, "version": 1}
        # deterministic mode is bit-identical to the ascending-rank fold
        assert o["det"].tobytes() == o["canon"].tobytes()
        np.testing.assert_allclose(o["fast"], o["canon"], rtol=1e-15)
        np.testing.assert_array_equal(o["bcast"], np.full(3, 7.0))
        np.testing.assert_array_equal(o["inplace"], np.full(4, 3.0))
        assert "mismatch" in o["mismatch"]
    assert res[0]["det"].tobytes() == res[1]["det"].tobytes()
    assert res[0]["part"] == (0, 500_000) and res[1]["part"] == (500_000, 1_000_000)
