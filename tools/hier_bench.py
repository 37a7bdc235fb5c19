"""Two-level CoCoA across GPUs on the C2 workload (torchrun, one rank per
(node, device)): the paper's hierarchy (K nodes x L devices, t2 inner rounds,
PAPER.md:68-69, 245-246) mapped onto one box's GPUs.  For each (K, L, t2)
with K * L = world: epochs per second (one epoch = one local pass per device;
an outer round has t2 of them) and inner rounds (epochs) to the 1e-3 duality
gap, eager rounds timed with CUDA events, max over ranks.  Rank 0 prints one
JSON line per topology.

    python -m torch.distributed.run --nproc-per-node 4 tools/hier_bench.py
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200.comm import NcclReducer, shutdown  # noqa: E402
from paper_1803_06333_b200.data import DeviceMatrix, partition_bounds  # noqa: E402

world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, bench.N_EX, bench.D_FEAT)
topologies = [(K, world // K, t2) for K in (world, world // 2, 1) if K >= 1 and world % K == 0
              for t2 in ((1,) if K == world else (1, 2))]
seen = set()
for K, L, t2 in topologies:
    if (K, L, t2) in seen or K * L != world:
        continue
    seen.add((K, L, t2))
    node, dev = divmod(rank, L)
    groups = [dist.new_group(list(range(k * L, (k + 1) * L))) for k in range(K)]
    b = partition_bounds(bench.N_EX, K, L)
    lo, hi = int(b[rank]), int(b[rank + 1])
    # this rank's examples (columns lo..hi of the 1M): whole generator blocks
    blo, bhi = lo // bench.BLOCK, -(-hi // bench.BLOCK)
    indptr, rows, vals, _ = bench.gen_columns(blo, bhi)
    off = lo - blo * bench.BLOCK
    ip = indptr[off:off + (hi - lo) + 1]
    dm = DeviceMatrix.from_csc(bench.D_FEAT, ip - ip[0], rows[ip[0]:ip[-1]], vals[ip[0]:ip[-1]])
    cfg = g.HierarchyConfig(nodes=K, devices=L, t2=t2, t1=10 ** 6, seed=0, epochs=1)
    eng = g.Engine(dm, spec, cfg, reducer=NcclReducer(), node_index=node,
                   device_index=dev if L > 1 or t2 > 1 else None,
                   node_reducer=NcclReducer(group=groups[node], deterministic=True),
                   n_total=bench.N_EX, mode="async", sync_solves=False, retry_budget=0,
                   cache_flags=1, peer_exchange=False)
    for _ in range(2):                 # warm-up: lazy NCCL communicators of the node groups
        eng.outer_round()
    eng.check_solves()
    eng.reset()
    obj, gap = eng.objective_and_gap()
    rounds, ms = 0, []
    while gap > 1e-3 * abs(obj) and rounds < 60:
        dist.barrier()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.outer_round()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(e)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms.append(float(t.item()))
        rounds += 1
        obj, gap = eng.objective_and_gap()
    eng.check_solves()
    if rank == 0:
        per_round = float(np.median(ms[1:])) if len(ms) > 1 else ms[0]
        print(json.dumps({"config": "C2 two-level", "n_gpus": world, "nodes": K, "devices": L,
                          "t2": t2, "outer_rounds_to_1e-3": rounds,
                          "epochs_to_1e-3": rounds * t2, "ms_per_outer_round": per_round,
                          "epochs_per_s": 1000.0 * t2 / per_round,
                          "time_to_target_ms": float(np.sum(ms)),
                          "timer": "eager rounds, CUDA events, max over ranks (gap checks excluded)",
                          "exchange": "NCCL (node all-gather per inner round, all-reduce per "
                                      "outer round)"}), flush=True)
    eng.close()
    del eng, dm
    torch.cuda.empty_cache()
sys.stdout.flush()
shutdown()
