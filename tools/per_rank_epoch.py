"""The per-GPU share of the C2 round at N = 1 / 2 / 4 / 8 on one GPU: the
first 8/N of bench.py's example blocks (1M / 500k / 250k / 125k examples,
the partition one rank owns at N GPUs), the bench's engine (async, one
attempt per round, fused turn without peers), rounds replayed from a CUDA
graph; step and epoch ms.  Used to project the 8-GPU step (this step plus
the peer part of the turn measured at 2 and 4 GPUs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200.data import DeviceMatrix

torch.cuda.set_device(0)
SHARES = [int(x) for x in os.environ.get("SHARES", "1,2,4,8").split(",")]
TRAJ = int(os.environ.get("TRAJ", "20"))
for n_gpus in SHARES:
    blocks = (bench.N_EX // bench.BLOCK) // n_gpus
    indptr, rows, vals, y = bench.gen_columns(0, blocks)
    dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
    spec = g.ObjectiveSpec("dual_l2_logistic", bench.LAM, bench.N_EX, bench.D_FEAT)
    eng = g.Engine(dm, spec, g.HierarchyConfig(nodes=1, t1=10 ** 6, seed=0, epochs=1),
                   mode="async", sync_solves=False, retry_budget=0, cache_flags=1)
    for _ in range(3):
        eng.outer_round()
    wk = next(iter(eng.workers.values()))
    traj = TRAJ
    eng.reset()
    graph = eng.capture(traj)
    best = 1e9
    for _ in range(6):
        eng.reset()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / traj)
    del graph
    eng.reset()
    wk.solver.timing_read()
    wk.solver.timing(True)
    for _ in range(10):
        eng.outer_round()
    torch.cuda.synchronize()
    k_ms, k_n = wk.solver.timing_read()
    wk.solver.timing(False)
    print(json.dumps({"share_of_n_gpus": n_gpus, "examples": len(y), "traj": traj, "step_ms": best,
                      "epoch_ms": k_ms[1] / max(k_n, 1)}), flush=True)
    eng.close()
    del eng, dm
    torch.cuda.empty_cache()
