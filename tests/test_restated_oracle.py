"""The restated kinds (not in the reference: parity unpinned) — their CPU
oracle restatements are checked against independent solutions: closed forms,
scikit-learn and SciPy L-BFGS. The GPU kernels are then checked against this
oracle (tests/test_gpu_restated.py)."""

import numpy as np
import pytest
from scipy import optimize

import oracle
from oracle import OMatrix


def _examples(n, d, k, seed, dense_frac=None):
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.integers(0, d - k + 1, size=(n, k)), axis=1) + np.arange(k)
    vals = rng.standard_normal((n, k))
    X = np.zeros((n, d))
    X[np.arange(n)[:, None], rows] = vals
    return X, rng


def _csc_of(dense_cols):
    """CSC of a dense matrix whose COLUMNS are the coordinates."""
    d, n = dense_cols.shape
    indptr = [0]
    rows, vals = [], []
    for j in range(n):
        nz = np.flatnonzero(dense_cols[:, j])
        rows.extend(nz.tolist())
        vals.extend(dense_cols[nz, j].tolist())
        indptr.append(len(rows))
    return OMatrix(d, np.array(indptr), np.array(rows, np.int32), np.array(vals))


def test_dual_ridge_matches_closed_form():
    X, rng = _examples(150, 20, 6, 1)
    y = X @ rng.standard_normal(20) + 0.1 * rng.standard_normal(150)
    lam = 0.7
    A = _csc_of(X.T)                         # columns = examples x_i (no label fold)
    r = oracle.train(A, "dual_ridge", lam, y=y, rounds=300, epochs=2, seed=1)
    w = r["v"] / lam
    w_star = np.linalg.solve(X.T @ X + lam * np.eye(20), X.T @ y)
    np.testing.assert_allclose(w, w_star, atol=1e-7)
    assert r["gap"][-1] < 1e-9 and np.all(np.diff(r["objective"]) <= 1e-12)


def test_elastic_net_matches_sklearn():
    from sklearn.linear_model import ElasticNet
    X, rng = _examples(200, 30, 8, 2)
    coef = rng.standard_normal(30) * (rng.random(30) < 0.5)
    b = X @ coef + 0.1 * rng.standard_normal(200)
    lam, rho = 3.0, 0.6
    A = _csc_of(X)                           # columns = features
    r = oracle.train(A, "elastic_net_primal", lam, target=b, rho=rho, rounds=800, epochs=2,
                     seed=3)
    sk = ElasticNet(alpha=lam / 200, l1_ratio=rho, fit_intercept=False, tol=1e-14,
                    max_iter=200000).fit(X, b)
    np.testing.assert_allclose(r["alpha"], sk.coef_, atol=1e-6)
    assert r["gap"][-1] < 1e-8
    # rho = 1 is exactly lasso
    la = oracle.train(A, "lasso_primal", lam, target=b, rounds=5, seed=3, record_gap=False)
    en = oracle.train(A, "elastic_net_primal", lam, target=b, rho=1.0, rounds=5, seed=3,
                      record_gap=False)
    np.testing.assert_array_equal(la["alpha"], en["alpha"])


def test_logistic_primal_matches_lbfgs_and_the_dual():
    X, rng = _examples(300, 25, 6, 3)
    y = np.where(X @ rng.standard_normal(25) + 0.3 * rng.standard_normal(300) >= 0, 1.0, -1.0)
    lam = 1.5
    A = _csc_of(X)
    r = oracle.train(A, "logistic_primal", lam, target=y, rounds=600, epochs=2, seed=4)

    def fg(w):
        z = y * (X @ w)
        val = 0.5 * lam * w @ w + np.sum(np.logaddexp(0.0, -z))
        s = -y * 0.5 * (1.0 + np.tanh(0.5 * -z))
        return val, lam * w + X.T @ s

    ref = optimize.minimize(fg, np.zeros(25), jac=True, method="L-BFGS-B",
                            options={"maxiter": 5000, "ftol": 1e-15, "gtol": 1e-12})
    np.testing.assert_allclose(r["alpha"], ref.x, atol=1e-6)
    assert r["objective"][-1] == pytest.approx(ref.fun, rel=1e-10)
    assert r["gap"][-1] < 1e-8
    # the dual kind on the label-folded examples reaches the same weights (w = v / lam)
    Ad = _csc_of((X * y[:, None]).T)
    rd = oracle.train(Ad, "dual_l2_logistic", lam, rounds=600, epochs=2, seed=4)
    np.testing.assert_allclose(rd["v"] / lam, ref.x, atol=1e-6)


def test_squared_hinge_primal_matches_lbfgs():
    X, rng = _examples(250, 15, 5, 5)
    y = np.where(X @ rng.standard_normal(15) >= 0, 1.0, -1.0)
    lam = 0.8
    A = _csc_of(X)
    r = oracle.train(A, "squared_hinge_primal", lam, target=y, rounds=800, epochs=2, seed=6)

    def fg(w):
        m = np.maximum(0.0, 1.0 - y * (X @ w))
        return 0.5 * lam * w @ w + 0.5 * m @ m, lam * w - X.T @ (y * m)

    ref = optimize.minimize(fg, np.zeros(15), jac=True, method="L-BFGS-B",
                            options={"maxiter": 5000, "ftol": 1e-15, "gtol": 1e-12})
    np.testing.assert_allclose(r["alpha"], ref.x, atol=1e-6)
    assert r["gap"][-1] < 1e-8


def _hinge_problem():
    X, rng = _examples(240, 12, 5, 9)
    y = np.where(X @ rng.standard_normal(12) + 0.2 * rng.standard_normal(240) >= 0, 1.0, -1.0)
    return X, y


@pytest.mark.parametrize("mu", [1.0, 0.3])
def test_smoothed_hinge_primal_matches_lbfgs(mu):
    """hinge_primal (smoothed hinge of width mu; the oracle's target is y / mu)
    against L-BFGS on the same smooth objective, with a certified gap."""
    X, y = _hinge_problem()
    lam = 0.5
    A = _csc_of(X)
    r = oracle.train(A, "hinge_primal", lam, target=y / mu, rounds=4000, epochs=2, seed=8)

    def fg(w):
        z = y * (X @ w)
        h = np.where(z >= 1, 0.0, np.where(z > 1 - mu, (1 - z) ** 2 / (2 * mu), 1 - z - mu / 2))
        dh = np.where(z >= 1, 0.0, np.where(z > 1 - mu, -(1 - z) / mu, -1.0))
        return 0.5 * lam * w @ w + h.sum(), lam * w + X.T @ (y * dh)

    ref = optimize.minimize(fg, np.zeros(12), jac=True, method="L-BFGS-B",
                            options={"maxiter": 20000, "ftol": 1e-15, "gtol": 1e-12})
    assert r["objective"][-1] == pytest.approx(ref.fun, rel=1e-8)
    np.testing.assert_allclose(r["alpha"], ref.x, atol=1e-4)
    assert r["gap"][-1] < 1e-9 * abs(r["objective"][-1])
    assert np.all(np.diff(r["objective"]) <= 1e-12 * abs(r["objective"][0]))


def test_smoothed_hinge_tends_to_the_hinge_svm():
    """mu -> 0 is the hinge-loss SVM.  Its optimum comes from the reference
    kind dual_l2_svm on the label-folded examples (a certified gap < 1e-8:
    hinge* = -F_dual*); the hinge objective of the smoothed solution lies in
    [hinge*, hinge* + n mu / 2 + its certified gap], a bracket that closes as
    mu shrinks."""
    X, y = _hinge_problem()
    lam = 0.5
    Ad = _csc_of((X * y[:, None]).T)
    rd = oracle.train(Ad, "dual_l2_svm", lam, rounds=3000, epochs=2, seed=8)
    assert rd["gap"][-1] < 1e-8
    hinge_star = -rd["objective"][-1]
    A = _csc_of(X)

    def hinge_obj(w):
        return 0.5 * lam * w @ w + np.maximum(0.0, 1.0 - y * (X @ w)).sum()

    # the primal of the dual solution is the hinge optimum itself
    assert hinge_obj(rd["v"] / lam) == pytest.approx(hinge_star, rel=1e-7)
    excess = []
    for mu in (1.0, 0.3, 0.1):
        r = oracle.train(A, "hinge_primal", lam, target=y / mu, rounds=4000, epochs=2, seed=8)
        f_mu = hinge_obj(r["alpha"])
        assert hinge_star - 1e-7 <= f_mu <= hinge_star + 0.5 * len(y) * mu + r["gap"][-1], mu
        excess.append(f_mu - hinge_star)
    assert excess[0] > excess[1] > excess[2]


def test_restated_steps_minimise_their_1d_models():
    rng = np.random.default_rng(7)
    for _ in range(200):
        ga, c, t, y = rng.standard_normal(), rng.uniform(0.1, 3), rng.standard_normal(), \
            rng.standard_normal()
        lam, rho = rng.uniform(0.1, 2), rng.uniform(0, 1)
        cases = {
            "dual_ridge": lambda s: ga * s + 0.5 * c * s * s + 0.5 * (t + s) ** 2 - y * (t + s),
            "elastic_net_primal": lambda s: ga * s + 0.5 * c * s * s
            + lam * (rho * abs(t + s) + 0.5 * (1 - rho) * (t + s) ** 2),
            "logistic_primal": lambda s: ga * s + 0.5 * c * s * s + 0.5 * lam * (t + s) ** 2,
        }
        for kind, phi in cases.items():
            rows = np.array([0], np.int32)
            vals = np.array([1.0])
            view = np.array([ga])
            step = oracle.coordinate_update(kind, lam, rows, vals, c, t, view, 1.0, rho=rho, y=y)
            best = optimize.minimize_scalar(phi, bounds=(-50, 50), method="bounded",
                                            options={"xatol": 1e-12}).x
            assert phi(step) <= phi(best) + 1e-10, kind
