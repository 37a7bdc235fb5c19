"""GPU parity of the dense column-major layout (C1 ridge, C3 HIGGS-shaped SVM):
the narrow-column kernels (d <= 1024: register-resident sequential warp,
CTA-replica asynchronous kernel) and the wide dense path, vs the CPU oracle
run on the same matrix in CSC form."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402


def _higgs(n, d, seed):
    """Dense examples normalised per row, labels from a planted w (SURVEY §8(d)
    C3), columns = label-folded examples (cli.py:173-181)."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal(d)
    X = rng.standard_normal((n, d))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    y = np.where(X @ w + 0.3 * rng.standard_normal(n) >= 0, 1.0, -1.0)
    return (X * y[:, None]).T.copy()          # (d, n): column i = y_i x_i


def _csc(dense):
    d, n = dense.shape
    indptr = np.arange(0, n * d + 1, d, dtype=np.int64)
    rows = np.tile(np.arange(d, dtype=np.int32), n)
    return oracle.OMatrix(d, indptr, rows, dense.T.reshape(-1).copy())


@pytest.mark.parametrize("d", [28, 60, 200, 500, 900])
def test_narrow_dense_sequential_matches_oracle(d):
    A = _higgs(3_000, d, d)
    m = g.DenseColumnMatrix(A)
    om = _csc(A)
    for kind, k in (("dual_l2_svm", 1), ("dual_l2_logistic", 0)):
        spec = g.ObjectiveSpec(kind, 5.0, m.n_cols, m.n_rows)
        for K in (1, 3):
            cfg = g.HierarchyConfig(nodes=K, t1=3, seed=2, epochs=2)
            res = g.train(m, spec, cfg, g.StoppingCriteria(max_rounds=3))
            want = oracle.train(om, k, 5.0, nodes=K, epochs=2, seed=2, rounds=3)
            np.testing.assert_allclose(res.trace.objectives(), want["objective"], rtol=1e-10)
            np.testing.assert_allclose(res.model.alpha, want["alpha"], atol=1e-7)


def test_wide_dense_ridge_c1_shape():
    """C1 restated as ridge_primal on dense data: coordinates = 120 features,
    d = 4000 examples (the wide dense path, view in shared memory)."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((4_000, 120)) / np.sqrt(120)
    b = X @ rng.standard_normal(120) + 0.1 * rng.standard_normal(4_000)
    m = g.DenseColumnMatrix(X)
    om = _csc(X)
    spec = g.ObjectiveSpec("ridge_primal", 1.0, 4_000, 120, target=b)
    res = g.train(m, spec, g.HierarchyConfig(t1=4, seed=1, epochs=1),
                  g.StoppingCriteria(max_rounds=4))
    want = oracle.train(om, 2, 1.0, target=b, epochs=1, seed=1, rounds=4)
    np.testing.assert_allclose(res.trace.objectives(), want["objective"], rtol=1e-10)
    np.testing.assert_allclose(res.trace.gaps(), want["gap"], rtol=1e-6, atol=1e-9)


def _epochs_to(gaps, objs, tol):
    """First round whose certified gap is <= tol * |F| (no division: F is 0
    at alpha = 0 for the SVM dual)."""
    hit = np.flatnonzero(np.asarray(gaps) <= tol * np.abs(np.asarray(objs)))
    return int(hit[0]) if len(hit) else None


@pytest.mark.parametrize("lam", [50.0, 500.0])
def test_narrow_dense_async_reaches_target_like_sequential(lam):
    """North-star async bar: the async run reaches the deterministic run's
    duality-gap target within the same number of epochs +-10% (two-sided; at
    least one epoch of slack for the integer granularity of a few-epoch
    count)."""
    A = _higgs(200_000, 28, 9)
    m = g.DenseColumnMatrix(A)
    spec = g.ObjectiveSpec("dual_l2_svm", lam, m.n_cols, m.n_rows)
    runs = {}
    for mode in ("sequential", "async"):
        eng = g.Engine(m, spec, g.HierarchyConfig(t1=12, seed=4, epochs=1), mode=mode)
        res = eng.train(g.StoppingCriteria(max_rounds=12))
        runs[mode] = _epochs_to(res.trace.gaps(), res.trace.objectives(), 1e-3)
    assert runs["sequential"] is not None and runs["async"] is not None, runs
    assert abs(runs["async"] - runs["sequential"]) <= max(1, round(0.1 * runs["sequential"])), \
        runs


def test_narrow_dense_async_delta_v_consistent():
    A = _higgs(50_000, 28, 5)
    m = g.DenseColumnMatrix(A)
    om = _csc(A)
    spec = g.ObjectiveSpec("dual_l2_svm", 20.0, m.n_cols, m.n_rows)
    lin = np.zeros(28)
    sub = g.LocalSubproblem(spec=spec, lin=lin, quad=1 / 20.0, const=0.0,
                            base=spec.init_alpha(), data=m, col_ids=np.arange(m.n_cols))
    res = g.damped_solve(sub, g.PermutationGenerator(3), 3, n_threads=8)
    assert res.final_subproblem_value < res.initial_subproblem_value
    assert np.all(np.diff(res.epoch_values) <= 0)
    dv = oracle.matvec(om, np.asarray(res.delta_alpha))
    assert np.max(np.abs(np.asarray(res.delta_v) - dv)) < 1e-9 * max(1.0, np.max(np.abs(dv)))


@pytest.mark.parametrize("d", [500, 900])
def test_narrow_async_wide_views(d):
    """16 / 32 view rows per lane (C1 dual's 500-row view): the async replica
    kernel keeps Delta v = B delta and decreases the subproblem."""
    A = _higgs(20_000, d, d + 1)
    m = g.DenseColumnMatrix(A)
    om = _csc(A)
    spec = g.ObjectiveSpec("dual_l2_svm", 5.0, m.n_cols, m.n_rows)
    sub = g.LocalSubproblem(spec=spec, lin=np.zeros(d), quad=1 / 5.0, const=0.0,
                            base=spec.init_alpha(), data=m, col_ids=np.arange(m.n_cols))
    res = g.damped_solve(sub, g.PermutationGenerator(4), 3, n_threads=8)
    assert res.final_subproblem_value < res.initial_subproblem_value
    assert np.all(np.diff(res.epoch_values) <= 0)
    dv = oracle.matvec(om, np.asarray(res.delta_alpha))
    assert np.max(np.abs(np.asarray(res.delta_v) - dv)) < 1e-9 * max(1.0, np.max(np.abs(dv)))


def test_narrow_dual_ridge_async_reaches_target_like_sequential():
    """C1 as BASELINE words it (ridge in the dual), scaled down: 6000 examples
    x 200 features, coordinates = examples on the narrow replica kernel. The
    async run reaches the deterministic run's 1e-3 gap target within +-10 %
    epochs."""
    rng = np.random.default_rng(12)
    n_ex, n_feat = 6_000, 200
    X = rng.standard_normal((n_ex, n_feat)) / np.sqrt(n_feat)
    b = X @ rng.standard_normal(n_feat) + 0.1 * rng.standard_normal(n_ex)
    m = g.DenseColumnMatrix(X.T)                        # column j = example j
    spec = g.ObjectiveSpec("dual_ridge", 1.0, n_ex, n_feat, target=b)
    runs = {}
    for mode in ("sequential", "async"):
        eng = g.Engine(m, spec, g.HierarchyConfig(t1=30, seed=3, epochs=1), mode=mode)
        res = eng.train(g.StoppingCriteria(max_rounds=30))
        runs[mode] = _epochs_to(res.trace.gaps(), res.trace.objectives(), 1e-3)
    assert runs["sequential"] is not None and runs["async"] is not None, runs
    assert abs(runs["async"] - runs["sequential"]) <= max(1, round(0.1 * runs["sequential"])), \
        runs
