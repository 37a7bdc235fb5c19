"""torchrun helper for tests/test_gpu_exchange.py: per-rank CoCoA node with the
peer-memory exchange vs the deterministic NCCL reducer (canonical_sum)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200.comm import NcclReducer  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    rng = np.random.default_rng(4)
    n, d, k = 30_000, 3_000, 10
    rows = np.sort(rng.integers(0, d - k + 1, size=(n, k)), axis=1) + np.arange(k)
    vals = rng.standard_normal((n, k))
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    vals *= np.where(rng.standard_normal(n) >= 0, 1.0, -1.0)[:, None]
    m = g.SparseColumnMatrix(d, np.arange(0, n * k + 1, k, dtype=np.int64),
                             rows.reshape(-1).astype(np.int32), vals.reshape(-1))
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, n, d)
    cfg = g.HierarchyConfig(nodes=world, t1=5, seed=9, epochs=1)
    res = []
    for peer, budget in ((False, 4), (True, 4), (True, 0)):
        eng = g.Engine(m, spec, cfg, reducer=NcclReducer(deterministic=True), node_index=rank,
                       mode="sequential", sync_solves=False, retry_budget=budget,
                       peer_exchange=peer)
        assert (eng.exchange is not None) == peer
        res.append(eng.train(g.StoppingCriteria(max_rounds=5)))
    o0, o1 = res[0].trace.objectives(), res[1].trace.objectives()
    for r in res[1:]:
        assert np.array_equal(o0, r.trace.objectives()), (o0, r.trace.objectives())
        assert np.array_equal(res[0].v, r.v)
        assert np.array_equal(res[0].model.alpha, r.model.alpha)
    ref = g.train(m, spec, cfg, g.StoppingCriteria(max_rounds=5))     # in-process K nodes
    assert np.allclose(o1, ref.trace.objectives(), rtol=1e-12, atol=0), (o1, ref.trace.objectives())
    if rank == 0:
        print("EXCHANGE OK", o1[-1], flush=True)
    sys.stdout.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
