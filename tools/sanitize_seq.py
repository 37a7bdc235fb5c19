"""Small deterministic and asynchronous solves for compute-sanitizer
(memcheck / racecheck / synccheck): the level-scheduled sequential kernel
(shared-memory view and L2 view), the one-warp walk, the narrow dense kernels,
the async kernel and the fused round turn."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_06333_b200 as g  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)


def sparse(n, d, k):
    rows = np.sort(rng.integers(0, d - k + 1, size=(n, k)), axis=1) + np.arange(k)
    vals = rng.standard_normal((n, k))
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    return g.SparseColumnMatrix(d, np.arange(0, n * k + 1, k, dtype=np.int64),
                                rows.reshape(-1).astype(np.int32), vals.reshape(-1))


for n, d in ((3000, 500), (4000, 20000)):
    m = sparse(n, d, 12)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, n, d)
    for mode in ("sequential", "async"):
        eng = g.Engine(m, spec, g.HierarchyConfig(t1=3, seed=1, epochs=1), mode=mode,
                       sync_solves=False, retry_budget=0)
        eng.train(g.StoppingCriteria(max_rounds=3))
        eng.close()
os.environ["GLM_SEQ_KERNEL"] = "csc"
m = sparse(2000, 800, 10)
g.train(m, g.ObjectiveSpec("dual_l2_svm", 1.0, 2000, 800), g.HierarchyConfig(t1=2, seed=2),
        g.StoppingCriteria(max_rounds=2))
os.environ.pop("GLM_SEQ_KERNEL")
A = rng.standard_normal((5000, 28))
A /= np.linalg.norm(A, axis=1, keepdims=True)
dm = g.DenseColumnMatrix(A.T)
spec = g.ObjectiveSpec("dual_l2_svm", 50.0, 5000, 28)
for mode in ("sequential", "async"):
    g.Engine(dm, spec, g.HierarchyConfig(t1=2, seed=4), mode=mode).train(
        g.StoppingCriteria(max_rounds=2))
torch.cuda.synchronize()
print("SANITIZE RUN OK")
