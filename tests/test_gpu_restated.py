"""GPU parity for the restated kinds vs the CPU oracle (which
tests/test_restated_oracle.py pins against closed forms / sklearn / SciPy)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402


def _problem(kind, seed=0, n=300, d=40, k=6):
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.integers(0, d - k + 1, size=(n, k)), axis=1) + np.arange(k)
    vals = rng.standard_normal((n, k))
    X = np.zeros((n, d))
    X[np.arange(n)[:, None], rows] = vals
    y = np.where(X @ rng.standard_normal(d) + 0.3 * rng.standard_normal(n) >= 0, 1.0, -1.0)
    if kind == "dual_ridge":
        cols, tgt = X.T, X @ rng.standard_normal(d) + 0.1 * rng.standard_normal(n)
        spec = g.ObjectiveSpec(kind, 0.7, n, d, target=tgt)
    elif kind == "elastic_net_primal":
        cols, tgt = X, X @ rng.standard_normal(d) + 0.1 * rng.standard_normal(n)
        spec = g.ObjectiveSpec(kind, 2.0, n, d, target=tgt, l1_ratio=0.6)
    elif kind == "hinge_primal":
        cols, tgt = X, y
        spec = g.ObjectiveSpec(kind, 1.2, n, d, target=tgt, smoothing=0.25)
    else:
        cols, tgt = X, y
        spec = g.ObjectiveSpec(kind, 1.2, n, d, target=tgt)
    nz = [np.flatnonzero(cols[:, j]) for j in range(cols.shape[1])]
    indptr = np.concatenate([[0], np.cumsum([len(z) for z in nz])])
    m = g.SparseColumnMatrix(cols.shape[0], indptr, np.concatenate(nz).astype(np.int32),
                             np.concatenate([cols[z, j] for j, z in enumerate(nz)]))
    return m, spec


KINDS = ["dual_ridge", "elastic_net_primal", "logistic_primal", "squared_hinge_primal",
         "hinge_primal"]


@pytest.mark.parametrize("kind", KINDS)
def test_engine_trace_vs_oracle(kind):
    m, spec = _problem(kind)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    kw = dict(target=spec.row_target, y=spec.coord_target, rho=spec.l1_ratio)
    for K, L, t2 in [(1, 1, 1), (2, 2, 2)]:
        ref = oracle.train(om, kind, spec.lam, nodes=K, devices=L, t2=t2, epochs=2, seed=5,
                           rounds=8, **kw)
        res = g.train(m, spec, g.HierarchyConfig(nodes=K, devices=L, t1=8, t2=t2, epochs=2,
                                                 seed=5), g.StoppingCriteria(max_rounds=8))
        np.testing.assert_allclose(res.trace.objectives(), ref["objective"], rtol=1e-10)
        gaps = np.array([r.gap for r in res.trace.rows], dtype=float)
        np.testing.assert_allclose(gaps, ref["gap"], rtol=1e-6, atol=1e-9)
        np.testing.assert_allclose(res.model.alpha, ref["alpha"], atol=1e-8)


@pytest.mark.parametrize("kind", KINDS)
def test_fused_round_vs_oracle(kind):
    """One attempt per round ending in the fused round turn (value, damping
    decision, Delta v exchange, next round's model in one kernel): the same
    bits as the unfused rounds and the oracle's trace, for every restated kind
    (their f terms run inside the turn's P1 and P3)."""
    m, spec = _problem(kind, seed=2)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    kw = dict(target=spec.row_target, y=spec.coord_target, rho=spec.l1_ratio)
    cfg = g.HierarchyConfig(t1=6, seed=7, epochs=1)
    runs = []
    for peer in (False, True):
        eng = g.Engine(m, spec, cfg, mode="sequential", sync_solves=False, retry_budget=0,
                       peer_exchange=peer)
        assert (eng.exchange is not None) == peer
        runs.append(eng.train(g.StoppingCriteria(max_rounds=6)))
        eng.close()
    np.testing.assert_array_equal(runs[0].trace.objectives(), runs[1].trace.objectives())
    np.testing.assert_array_equal(runs[0].model.alpha, runs[1].model.alpha)
    np.testing.assert_array_equal(runs[0].v, runs[1].v)
    ref = oracle.train(om, kind, spec.lam, epochs=1, seed=7, rounds=6, **kw)
    np.testing.assert_allclose(runs[1].trace.objectives(), ref["objective"], rtol=1e-10)


@pytest.mark.parametrize("kind", KINDS)
def test_damped_solve_vs_oracle(kind):
    m, spec = _problem(kind, seed=1)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    alpha = spec.init_alpha()
    v = oracle.matvec(om, alpha)
    lin = oracle.f_grad(kind, spec.lam, spec.row_target, v)
    fv = oracle.f_eval(kind, spec.lam, spec.row_target, v)
    sub = g.LocalSubproblem(spec=spec, lin=lin, quad=spec.beta * 1.5, const=fv, base=alpha,
                            data=m, col_ids=np.arange(m.n_cols))
    gen = g.PermutationGenerator(11)
    res = g.damped_solve(sub, gen, 3)
    want = oracle.damped_solve(kind, spec.lam, om, lin, spec.beta * 1.5, fv, alpha, 11, 3,
                               rho=spec.l1_ratio, y=spec.coord_target)
    assert res.epochs_run == want["epochs_run"] and gen.state == want["gen_state"]
    np.testing.assert_allclose(res.epoch_values, want["values"], rtol=1e-11)
    np.testing.assert_allclose(res.delta_alpha, want["delta"], atol=1e-9)
