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


def _hier_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1803_06333_b200.comm import NcclReducer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, L = 2, 2
        node, dev = divmod(rank, L)
        groups = [dist.new_group(list(range(k * L, (k + 1) * L))) for k in range(K)]
        node_red = NcclReducer(group=groups[node], deterministic=True)
        glob = NcclReducer(deterministic=True)
        rng = np.random.default_rng(5)
        dvs = rng.standard_normal((2, K, L, 64)) * 1e3      # [inner round, node, device]
        # Engine._run_node with one rank per device: v_bar += every device's
        # Delta v in device order, then the outer sum with one contribution per node
        vbar = torch.zeros(64, dtype=torch.float64)
        for t in range(2):
            for part in node_red.allgather(torch.from_numpy(dvs[t, node, dev].copy())):
                vbar += part
        total = vbar.clone() if dev == 0 else torch.zeros(64, dtype=torch.float64)
        glob.allreduce_inplace(total)
        q.put((rank, total.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_four_rank_hierarchical_fold():
    """K = 2 nodes x L = 2 devices as four gloo ranks: the node fold over an
    allgather plus the outer sum with one contribution per node equals the
    in-process nested fold (engine.py:259-282) bit for bit."""
    world = 4
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_hier_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dvs = np.random.default_rng(5).standard_normal((2, 2, 2, 64)) * 1e3
    total = np.zeros(64)
    for k in range(2):
        vbar = np.zeros(64)
        for t in range(2):
            for l in range(2):
                vbar = vbar + dvs[t, k, l]
        total = total + vbar
    for r in range(world):
        assert res[r].tobytes() == total.tobytes()
