"""Deterministic-mode epoch time on bench.py's C2 arrays: damped_solve
(n_threads=1) for 1 and 3 epochs; (t3 - t1) / 2 = one epoch incl. its value
check.  GLM_SEQ_KERNEL=csc selects the one-warp walk for comparison."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else bench.N_EX // bench.BLOCK
indptr, rows, vals, _ = bench.gen_columns(0, nb)
m = g.SparseColumnMatrix(bench.D_FEAT, indptr, rows, vals, validate=False)
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
alpha = spec.init_alpha()
v = m.matvec(alpha)
sub = g.LocalSubproblem(spec=spec, lin=v, quad=1.0, const=float(v @ v) / 2, base=alpha, data=m,
                        col_ids=np.arange(m.n_cols))
out = {}
for env in (None, "csc") if "--both" in sys.argv else (None,):
    if env:
        os.environ["GLM_SEQ_KERNEL"] = env
    ts = {}
    for ep in (1, 3):
        g.damped_solve(sub, g.PermutationGenerator(1), 1, n_threads=1)      # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = g.damped_solve(sub, g.PermutationGenerator(1), ep, n_threads=1)
        torch.cuda.synchronize()
        ts[ep] = time.perf_counter() - t0
    out[env or "levels"] = {"epoch_s": (ts[3] - ts[1]) / 2, "solve1_s": ts[1],
                            "final": res.final_subproblem_value}
    os.environ.pop("GLM_SEQ_KERNEL", None)
print(out)
