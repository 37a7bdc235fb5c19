"""torchrun helper for tests/test_gpu_exchange.py: per-rank CoCoA node with the
peer-memory exchange (csrc/peer.cu) vs the deterministic reducer
(canonical_sum, comm.py:41-46).

  (default)      one GPU per rank, NCCL process group
  --same-gpu     every rank on cuda:0, gloo process group (NCCL refuses two
                 ranks on one GPU): the flag / fence / parity protocol and the
                 IPC mappings are the same, the ranks' kernels time-slice
  --kill         rank 1 dies after two rounds; rank 0 must raise ReduceError
                 from the exchange's device-side deadline instead of hanging
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200.comm import NcclReducer, ReduceError, shutdown  # noqa: E402


def matrix(n=30_000, d=3_000, k=10, seed=4):
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.integers(0, d - k + 1, size=(n, k)), axis=1) + np.arange(k)
    vals = rng.standard_normal((n, k))
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    vals *= np.where(rng.standard_normal(n) >= 0, 1.0, -1.0)[:, None]
    return g.SparseColumnMatrix(d, np.arange(0, n * k + 1, k, dtype=np.int64),
                                rows.reshape(-1).astype(np.int32), vals.reshape(-1))


def parity(rank, world, m, modes):
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    cfg = g.HierarchyConfig(nodes=world, t1=5, seed=9, epochs=1)
    res = []
    for mode, peer, budget in ((modes[0], False, 4), (modes[0], True, 4), (modes[0], True, 0)):
        eng = g.Engine(m, spec, cfg, reducer=NcclReducer(deterministic=True), node_index=rank,
                       mode=mode, sync_solves=False, retry_budget=budget, peer_exchange=peer)
        assert (eng.exchange is not None) == peer, "peer exchange did not come up"
        res.append(eng.train(g.StoppingCriteria(max_rounds=5)))
        eng.close()
    o0 = res[0].trace.objectives()
    for r in res[1:]:
        assert np.array_equal(o0, r.trace.objectives()), (o0, r.trace.objectives())
        assert np.array_equal(res[0].v, r.v)
        assert np.array_equal(res[0].model.alpha, r.model.alpha)
    ref = g.train(m, spec, cfg, g.StoppingCriteria(max_rounds=5), mode=modes[0])  # in-process K
    assert np.allclose(o0, ref.trace.objectives(), rtol=1e-12, atol=0), (o0, ref.trace.objectives())
    if rank == 0:
        print("EXCHANGE OK", o0[-1], flush=True)
    # the benched configuration (async epoch kernel with L1-cached view
    # gathers, fused turn, CUDA-graph replay) across the ranks: a graph replay
    # equals the eager rounds bit for bit, and v = A alpha afterwards
    for mode in modes[1:]:
        eng = g.Engine(m, spec, cfg, reducer=NcclReducer(deterministic=True), node_index=rank,
                       mode=mode, sync_solves=False, retry_budget=0, cache_flags=1)
        assert eng.exchange is not None
        graph = eng.capture(4)
        eng.reset()
        graph.replay()
        torch.cuda.synchronize()
        eng.check_solves()
        v_graph, a_graph = eng.v, eng.alpha_global()
        if mode == "sequential":          # deterministic: replay == eager rounds, bitwise
            eng.reset()
            for _ in range(4):
                eng.outer_round()
            eng.check_solves()
            assert np.array_equal(eng.v, v_graph) and np.array_equal(eng.alpha_global(), a_graph)
        from oracle import OMatrix, matvec
        want = matvec(OMatrix(m.n_rows, m.indptr, m.rows, m.vals), a_graph)
        err = np.max(np.abs(v_graph - want))
        assert err <= 1e-9 * max(1.0, np.max(np.abs(want))), err
        del graph
        eng.close()
        if rank == 0:
            print(f"GRAPH {mode} OK v=A.alpha err {err:.3g}", flush=True)


def kill(rank, world, m):
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    cfg = g.HierarchyConfig(nodes=world, t1=5, seed=9, epochs=1)
    eng = g.Engine(m, spec, cfg, reducer=NcclReducer(deterministic=True), node_index=rank,
                   mode="async", sync_solves=False, retry_budget=0, peer_timeout=3.0)
    assert eng.exchange is not None
    for _ in range(2):
        eng.outer_round()
    eng.check_solves()
    dist.barrier()
    if rank == 1:
        sys.stdout.flush()
        os._exit(0)          # dies without publishing its next Delta v
    try:
        for _ in range(2):
            eng.outer_round()
        eng.check_solves()
    except ReduceError as exc:
        print("TIMEOUT OK", exc, flush=True)
        sys.stdout.flush()
        os._exit(0)          # the process group has a dead member: no teardown
    except Exception as exc:  # a CUDA error after the peer's memory went away
        print("TIMEOUT CUDA", repr(exc), flush=True)
        sys.stdout.flush()
        os._exit(0)
    print("NO ERROR: the surviving rank did not notice the dead peer", flush=True)
    sys.stdout.flush()
    os._exit(1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--same-gpu", action="store_true")
    ap.add_argument("--kill", action="store_true")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    if args.same_gpu:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    m = matrix()
    if args.kill:
        return kill(rank, world, m)
    if not args.same_gpu:      # NcclReducer's host-vector path (pinned and pageable)
        red = NcclReducer()
        for n in (100_003, 7):
            vecs = [np.random.default_rng(100 + r).standard_normal(n) for r in range(world)]
            want = vecs[0].copy()
            for r in range(1, world):
                want = want + vecs[r]
            pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
            pin[:] = vecs[rank]
            got = red.allreduce_sum(pin, out=pin)
            assert got is pin and np.array_equal(pin, want), "pinned host allreduce"
            got2 = red.allreduce_sum(vecs[rank].copy())
            assert np.array_equal(got2, want), "pageable host allreduce"
        if rank == 0:
            print("HOST ALLREDUCE OK", flush=True)
    parity(rank, world, m, ("sequential", "sequential", "async"))
    sys.stdout.flush()
    shutdown()


if __name__ == "__main__":
    main()
