"""GlmEstimator (estimator.ts / SPEC.md pybind surface): host-side contract on
CPU, fit/predict parity with the reference's own trained model on its bundled
dataset (tests/golden/predict.npz, made by running the reference) on the GPU."""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_1803_06333_b200.estimator import (GlmEstimator, NotFittedError, examples_matrix,
                                             normalize_labels)


def _tiny(golden):
    d = golden("data")
    X = sp.csr_matrix((d["ex_vals"], d["ex_rows"], d["ex_indptr"]),
                      shape=(len(d["ex_indptr"]) - 1, int(d["ex_n_rows"])))
    return X, d["ex_labels"]


# ------------------------------------------------------------------- CPU
def test_params_roundtrip_and_validation():
    est = GlmEstimator(objective="dual-svm", lam=0.5)
    p = est.get_params()
    assert p["objective"] == "dual-svm" and p["lam"] == 0.5 and p["max_rounds"] == 20
    assert est.set_params(epochs=3) is est and est.get_params()["epochs"] == 3
    with pytest.raises(ValueError):
        est.set_params(objective="kernel-svm")
    with pytest.raises(ValueError):
        GlmEstimator(lam=0.0)
    with pytest.raises(TypeError):
        GlmEstimator(alpha=1.0)
    assert not est.fitted
    with pytest.raises(NotFittedError):
        est.coefficients()
    with pytest.raises(NotFittedError):
        est.predict(np.zeros((2, 2)))


def test_label_normalisation_contract():
    np.testing.assert_array_equal(normalize_labels([0, 1, 1, 0]), [-1, 1, 1, -1])
    np.testing.assert_array_equal(normalize_labels([-1, 1]), [-1, 1])
    with pytest.raises(ValueError, match="binary"):
        normalize_labels([0, 1, 2])
    with pytest.raises(ValueError, match="mix"):
        normalize_labels([-1, 0, 1])


def test_examples_matrix_layouts_agree(golden):
    X, _ = _tiny(golden)
    a = examples_matrix(X)
    b = examples_matrix(X.toarray())
    rows = [[(int(j), float(v)) for j, v in zip(r.indices, r.data)] for r in X]
    c = examples_matrix(rows, n_features=X.shape[1])
    d = golden("data")
    for m in (a, b, c):
        np.testing.assert_array_equal(m.indptr, d["ex_indptr"])
        np.testing.assert_array_equal(m.rows, d["ex_rows"])
        np.testing.assert_array_equal(m.vals, d["ex_vals"])
    with pytest.raises(ValueError, match="increasing"):
        examples_matrix([[(1, 1.0), (0, 2.0)]])


# ------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("kind,obj", [("dual_l2_logistic", "dual-logistic"),
                                      ("dual_l2_svm", "dual-svm"), ("ridge_primal", "ridge")])
def test_fit_predict_matches_reference_model(golden, kind, obj):
    """Same hyper-parameters as the reference's trained model (gen_predict:
    lambda 0.5, t1 5, seed 3, 2 epochs, K = L = 1, 1 thread)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    z = golden("predict")
    X, y = _tiny(golden)
    est = GlmEstimator(objective=obj, lam=0.5, epochs=2, seed=3, max_rounds=5).fit(X, y)
    p = kind + "_"
    np.testing.assert_allclose([r["objective"] for r in est.trace_], z[p + "objective"],
                               rtol=1e-10)
    np.testing.assert_allclose(est.coefficients(), z[p + "w"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(est.decision_function(X), z[p + "scores"], rtol=1e-9,
                               atol=1e-12)
    if kind.startswith("dual_"):
        prob = est.predict_proba(X)
        assert np.max(np.abs(prob - z[p + "prob"])) < 1e-12
        np.testing.assert_array_equal(est.predict(X), np.where(z[p + "prob"] >= 0.5, 1, -1))
        ev = est.evaluate(X, y)
        assert ev["logloss"] == pytest.approx(float(z[p + "logloss"]), rel=1e-10)
        assert ev["accuracy"] == float(z[p + "accuracy"])
    else:
        assert -est.score(X, y) == pytest.approx(float(z[p + "mse"]), rel=1e-9)


@pytest.mark.gpu
def test_fit_separable_determinism_and_errors(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    X = np.array([[1.0, 0.2], [0.9, -0.1], [-1.0, 0.1], [-0.8, -0.3]])
    y = np.array([1, 1, 0, 0])
    est = GlmEstimator(objective="dual-svm", lam=0.1, max_rounds=30)
    np.testing.assert_array_equal(est.fit(X, y).predict(X), [1, 1, -1, -1])
    w1 = est.coefficients()
    np.testing.assert_array_equal(GlmEstimator(objective="dual-svm", lam=0.1,
                                               max_rounds=30).fit(X, y).coefficients(), w1)
    with pytest.raises(ValueError):
        est.predict(np.zeros((1, 3)))                     # more features than fitted
    with pytest.raises(ValueError):
        GlmEstimator().fit(X, [0, 1, 2, 1])               # three classes
    est.save(tmp_path / "m.bin")
    back = GlmEstimator.load(tmp_path / "m.bin")
    np.testing.assert_array_equal(back.coefficients(), w1)
    np.testing.assert_array_equal(back.predict(X), est.predict(X))
