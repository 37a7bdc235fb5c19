import sys, numpy as np
sys.path.insert(0, '.')
import oracle, paper_1803_06333_b200 as g
def _higgs(n, d, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal(d)
    X = rng.standard_normal((n, d))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    y = np.where(X @ w + 0.3 * rng.standard_normal(n) >= 0, 1.0, -1.0)
    return (X * y[:, None]).T.copy()
def _csc(dense):
    d, n = dense.shape
    indptr = np.arange(0, n * d + 1, d, dtype=np.int64)
    rows = np.tile(np.arange(d, dtype=np.int32), n)
    return oracle.OMatrix(d, indptr, rows, dense.T.reshape(-1).copy())
for d in (28, 60, 100, 200):
    A = _higgs(3000, d, d); m = g.DenseColumnMatrix(A); om = _csc(A)
    spec = g.ObjectiveSpec("dual_l2_svm", 5.0, m.n_cols, m.n_rows)
    for K in (1, 3):
        eng = g.Engine(m, spec, g.HierarchyConfig(nodes=K, t1=3, seed=2, epochs=2))
        objs = []
        for r in range(3):
            eng.outer_round(); objs.append(eng.objective_and_gap()[0])
        a = eng.alpha
        w = oracle.train(om, 1, 5.0, nodes=K, epochs=2, seed=2, rounds=3)
        print(d, K, "maxa-1", a.max() - 1, "dev", np.abs(a - w["alpha"]).max(),
              "obj", objs[-1], w["objective"][-1], flush=True)
