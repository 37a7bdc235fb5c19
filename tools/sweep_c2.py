"""Sweep scd_async launch shapes on the C2 workload (1M x 100k, 40 nnz).

Reports per-variant epoch-kernel time (CUDA events inside the library), the
permutation/value times, and epochs to a 1e-3 relative duality gap."""
import sys
import os
import json
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200.data import DeviceMatrix

torch.cuda.set_device(0)
indptr, rows, vals, y = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
spec = g.ObjectiveSpec("dual_l2_logistic", bench.LAM, bench.N_EX, bench.D_FEAT)
cfg = g.HierarchyConfig(t1=10 ** 6, seed=0, epochs=1)
import itertools
LANES = [int(x) for x in os.environ.get("SWEEP_LANES", "4,2564,1288,8").split(",")]
CMS = [int(x) for x in os.environ.get("SWEEP_CM", "1").split(",")]
variants = [dict(group_lanes=l, cache_flags=c) for c, l in itertools.product(CMS, LANES)]
out = []
for var in variants:
    eng = g.Engine(dm, spec, cfg, mode="async", sync_solves=False, retry_budget=0, **var)
    wk = next(iter(eng.workers.values()))
    for _ in range(5):
        eng.outer_round()
    torch.cuda.synchronize()
    wk.solver.timing(True)
    t0 = time.perf_counter()
    steps = 50
    for _ in range(steps):
        eng.outer_round()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e3
    ms, n = wk.solver.timing_read()
    wk.solver.timing(False)
    eng2 = g.Engine(dm, spec, cfg, mode="async", sync_solves=False, retry_budget=0, **var)
    obj, gap = eng2.objective_and_gap()
    r = 0
    while gap > 1e-3 * abs(obj) and r < 100:
        eng2.outer_round()
        r += 1
        obj, gap = eng2.objective_and_gap()
    rec = dict(var, step_ms=wall, perm_ms=ms[0] / n, epoch_ms=ms[1] / n, value_ms=ms[2] / n,
               epochs_to_1e3=r, gap=gap, obj=obj)
    print(json.dumps(rec), flush=True)
