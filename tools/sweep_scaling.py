"""Strong-scaling proxy on one GPU: the C2 problem split into K CoCoA nodes
in-process (exactly the math of K GPUs; the K solves run back to back here).
Reports per-node epoch-kernel time and epochs to a 1e-3 relative gap for the
in-flight caps given."""
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200.data import DeviceMatrix

torch.cuda.set_device(0)
indptr, rows, vals, y = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
spec = g.ObjectiveSpec("dual_l2_logistic", bench.LAM, bench.N_EX, bench.D_FEAT)
caps = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0"])]
Ks = [int(k) for k in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "4", "8"])]
for K, cap in itertools.product(Ks, caps):
    cfg = g.HierarchyConfig(nodes=K, t1=10 ** 6, seed=0, epochs=1)
    eng = g.Engine(dm, spec, cfg, mode="async", sync_solves=False, retry_budget=0,
                   group_lanes=4, cache_flags=1, max_inflight=cap)
    wk = eng.workers[(0, 0)]
    for _ in range(3):
        eng.outer_round()
    torch.cuda.synchronize()
    wk.solver.timing_read()
    wk.solver.timing(True)
    eng.reset()
    t0 = time.perf_counter()
    for _ in range(20):
        eng.outer_round()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 20 * 1e3
    ms, n = wk.solver.timing_read()
    wk.solver.timing(False)
    eng.reset()
    obj, gap = eng.objective_and_gap()
    r = 0
    while gap > 1e-3 * abs(obj) and r < 200:
        eng.outer_round()
        r += 1
        obj, gap = eng.objective_and_gap()
    print(json.dumps(dict(K=K, cap=cap, m=bench.N_EX // K, round_ms_all_nodes=wall,
                          perm_ms=ms[0] / n, epoch_ms=ms[1] / n, value_ms=ms[2] / n,
                          epochs_to_1e3=r)), flush=True)
