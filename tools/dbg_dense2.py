import sys, numpy as np
sys.path.insert(0, '.')
import oracle, paper_1803_06333_b200 as g
from paper_1803_06333_b200 import objectives
exec(open('tools/dbg_dense.py').read().split("for d in")[0].split("import oracle, paper_1803_06333_b200 as g")[1])
objectives.ObjectiveSpec.check_alpha = lambda self, a: None
for d in (28, 60, 200):
    A = _higgs(3000, d, d); m = g.DenseColumnMatrix(A); om = _csc(A)
    for kind, k in (("dual_l2_svm", 1), ("dual_l2_logistic", 0)):
        spec = g.ObjectiveSpec(kind, 5.0, m.n_cols, m.n_rows)
        for K in (1, 3):
            res = g.train(m, spec, g.HierarchyConfig(nodes=K, t1=3, seed=2, epochs=2), g.StoppingCriteria(max_rounds=3))
            w = oracle.train(om, k, 5.0, nodes=K, epochs=2, seed=2, rounds=3)
            a = res.model.alpha
            bad = np.flatnonzero((a > 1) | (a < 0))
            print(d, kind, K, "nbad", len(bad), a[bad[:3]] - 1 if len(bad) else "", w["alpha"][bad[:3]] if len(bad) else "",
                  "dev", np.abs(a - w["alpha"]).max(), "obj", res.trace.objectives()[-1] - w["objective"][-1], flush=True)
