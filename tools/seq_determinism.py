"""Bit-determinism of the deterministic mode at full C2 size: two solves of
each sequential kernel from the same state must agree bit for bit, and the
level-scheduled kernels must equal the one-warp walk."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else bench.N_EX // bench.BLOCK
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
indptr, rows, vals, _ = bench.gen_columns(0, nb)
m = g.SparseColumnMatrix(bench.D_FEAT, indptr, rows, vals, validate=False)
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
alpha = spec.init_alpha()
v = m.matvec(alpha)
sub = g.LocalSubproblem(spec=spec, lin=v, quad=1.0, const=float(v @ v) / 2, base=alpha, data=m,
                        col_ids=np.arange(m.n_cols))
out = {}
for env in ("csc", None):
    os.environ.pop("GLM_SEQ_KERNEL", None)
    if env:
        os.environ["GLM_SEQ_KERNEL"] = env
    runs = [g.damped_solve(sub, g.PermutationGenerator(1), epochs, n_threads=1) for _ in range(2)]
    out[env or "levels"] = runs
    same = all(np.asarray(r.delta_alpha).tobytes() == np.asarray(runs[0].delta_alpha).tobytes()
               and np.asarray(r.delta_v).tobytes() == np.asarray(runs[0].delta_v).tobytes()
               for r in runs)
    print(env or "levels", "repeatable:", same, repr(runs[0].final_subproblem_value),
          repr(runs[1].final_subproblem_value), flush=True)
ref = out["csc"][0]
for k in ("levels",):
    r = out[k][0]
    da = np.asarray(r.delta_alpha) - np.asarray(ref.delta_alpha)
    dv = np.asarray(r.delta_v) - np.asarray(ref.delta_v)
    print(k, "== csc:", not da.any() and not dv.any(), "coords differing:",
          int(np.count_nonzero(da)), "max |d delta|:", float(np.max(np.abs(da))),
          "rows differing:", int(np.count_nonzero(dv)), flush=True)
