"""torchrun helper for tests/test_gpu_exchange.py: the two-level scheme across
ranks — K nodes x L devices, one rank per (node, device), t2 inner rounds
with the node's Delta v folded over the node's ranks each inner round and
the nodes' v_bar summed over all ranks each outer round (engine.py:239-307)
— against the in-process engine with the same K x L x t2 (bit-identical in
the deterministic mode: the same additions in the same order).

  --nodes K --devices L   (world = K * L)
  --same-gpu              every rank on cuda:0, gloo process groups
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200.comm import NcclReducer, shutdown  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--devices", type=int, default=2)
    ap.add_argument("--t2", type=int, default=2)
    ap.add_argument("--same-gpu", action="store_true")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    K, L = args.nodes, args.devices
    assert world == K * L
    if args.same_gpu:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    node, dev = divmod(rank, L)
    groups = [dist.new_group(list(range(k * L, (k + 1) * L))) for k in range(K)]
    node_red = NcclReducer(group=groups[node], deterministic=True)
    rng = np.random.default_rng(12)
    n, d, k = 24_000, 2_000, 9
    rows = np.sort(rng.integers(0, d - k + 1, size=(n, k)), axis=1) + np.arange(k)
    vals = rng.standard_normal((n, k))
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    vals *= np.where(rng.standard_normal(n) >= 0, 1.0, -1.0)[:, None]
    m = g.SparseColumnMatrix(d, np.arange(0, n * k + 1, k, dtype=np.int64),
                             rows.reshape(-1).astype(np.int32), vals.reshape(-1))
    out = {}
    for kind in ("dual_l2_logistic", "dual_l2_svm"):
        spec = g.ObjectiveSpec(kind, 1.0, n, d)
        cfg = g.HierarchyConfig(nodes=K, devices=L, t1=4, t2=args.t2, seed=3, epochs=2)
        eng = g.Engine(m, spec, cfg, reducer=NcclReducer(deterministic=True), node_index=node,
                       device_index=dev, node_reducer=node_red, mode="sequential")
        res = eng.train(g.StoppingCriteria(max_rounds=4))
        ref = g.train(m, spec, cfg, g.StoppingCriteria(max_rounds=4), mode="sequential")
        o, o_ref = res.trace.objectives(), ref.trace.objectives()
        if kind == "dual_l2_svm":
            # alpha0 = 0, v0 = 0 exactly: alpha and v see the same additions in
            # the same order (the reported objective sums g over the ranks'
            # partial sums, so it agrees to rounding only)
            assert np.array_equal(res.v, ref.v)
            assert np.array_equal(res.model.alpha, ref.model.alpha)
            assert np.allclose(o, o_ref, rtol=1e-13, atol=0), (kind, o, o_ref)
        else:
            # v0 = A alpha0 is summed per rank, then across ranks (one SpMV
            # in-process): rounding-level differences only
            assert np.allclose(o, o_ref, rtol=1e-12, atol=0), (kind, o, o_ref)
            assert np.allclose(res.model.alpha, ref.model.alpha, rtol=0, atol=1e-9)
            assert np.allclose(res.v, ref.v, rtol=1e-10, atol=1e-12)
        g_ours = np.array([r.gap for r in res.trace.rows])
        g_ref = np.array([r.gap for r in ref.trace.rows])
        assert np.allclose(g_ours, g_ref, rtol=1e-9, atol=1e-12), (g_ours, g_ref)
        out[kind] = res.trace.objectives()[-1]
    # async per-rank solves: the fold is the same, only the epochs differ
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, n, d)
    cfg = g.HierarchyConfig(nodes=K, devices=L, t1=6, t2=args.t2, seed=3, epochs=1)
    eng = g.Engine(m, spec, cfg, reducer=NcclReducer(), node_index=node, device_index=dev,
                   node_reducer=node_red, mode="async")
    res = eng.train(g.StoppingCriteria(max_rounds=6))
    objs = res.trace.objectives()
    assert np.all(np.diff(objs) <= 1e-9 * np.abs(objs[1:])), objs
    from oracle import OMatrix, matvec
    want = matvec(OMatrix(d, m.indptr, m.rows, m.vals), res.model.alpha)
    assert np.max(np.abs(res.v - want)) <= 1e-9 * max(1.0, np.max(np.abs(want)))
    if rank == 0:
        print(f"HIER OK K={K} L={L} t2={args.t2}", out, flush=True)
    sys.stdout.flush()
    shutdown()


if __name__ == "__main__":
    main()
