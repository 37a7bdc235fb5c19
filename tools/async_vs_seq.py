"""North-star async contract at N GPUs (torchrun, one process per GPU): on the
C2 workload, rounds (1 epoch each) to duality gap <= 1e-3 |F| in the
deterministic sequential mode vs the asynchronous mode, same CoCoA
partitioning (K = N).  Rank 0 prints one JSON line.

`VIRTUAL_NODES=K` (one process): the K CoCoA nodes run one after another on
one GPU, each with the partition, permutation stream and kernel
configuration (in-flight coordinates) it would have on its own GPU — the
algorithm of K GPUs, e.g. K = 8 on a box with fewer."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200.comm import NcclReducer
from paper_1803_06333_b200.data import DeviceMatrix

world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
per = (bench.N_EX // bench.BLOCK) // world
indptr, rows, vals, y = bench.gen_columns(rank * per, (rank + 1) * per)
dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, bench.N_EX, bench.D_FEAT)
kw = dict(reducer=NcclReducer(), node_index=rank, n_total=bench.N_EX) if world > 1 else {}
K = int(os.environ.get("VIRTUAL_NODES", "0")) if world == 1 else 0
out = {"n_gpus": world, "target": "gap <= 1e-3 |F|"}
if K:
    out["virtual_nodes"] = K
for mode in ("sequential", "async"):
    eng = g.Engine(dm, spec, g.HierarchyConfig(nodes=K or world, t1=10**6, seed=0, epochs=1),
                   mode=mode, sync_solves=False, retry_budget=0, cache_flags=1, **kw)
    obj, gap = eng.objective_and_gap()
    rounds = 0
    while gap > 1e-3 * abs(obj) and rounds < 40:
        eng.outer_round()
        rounds += 1
        obj, gap = eng.objective_and_gap()
    out[mode] = {"rounds": rounds, "rel_gap": gap / abs(obj)}
if rank == 0:
    s, a = out["sequential"]["rounds"], out["async"]["rounds"]
    out["within_10pct"] = abs(a - s) <= max(1, 0.1 * s)
    print(json.dumps(out), flush=True)
sys.stdout.flush()
from paper_1803_06333_b200.comm import shutdown  # noqa: E402
shutdown()
