"""Estimator API: fit / predict / predict_proba / objective over the B200 engine.

Mirrors the reference's estimator surface — `GlmEstimator` (frontend/src/
estimator.ts:20-162: getParams/setParams, fit, predictProba, predict,
coefficients, trace) and the SPEC's pybind module (fit before
predict, binary labels {-1,+1} or {0,1} normalised internally, three classes
or mixed conventions rejected, feature-count mismatch rejected, fit twice with
the same seed gives identical coefficients) — in Python and in-process: the
TypeScript class drives `hierglm train/predict` through files, here the same
hyper-parameters drive the device-resident Engine directly and prediction
runs the fused scores / sigmoid kernel (modelio.py:57-99, cli.py:271-300).

Data layout follows load_training_data (cli.py:146-185): dual kinds train on
the label-folded examples as columns, primal kinds on the features as columns
with the labels as the regression target.
"""

from __future__ import annotations

import numpy as np

from . import modelio
from .data import SparseColumnMatrix
from .engine import Engine, HierarchyConfig, StoppingCriteria
from .objectives import ObjectiveSpec

# cli.py:20-25 names, plus the restated kinds of this package
OBJECTIVE_NAMES = {
    "dual-logistic": "dual_l2_logistic",
    "dual-svm": "dual_l2_svm",
    "ridge": "ridge_primal",
    "lasso": "lasso_primal",
    "dual-ridge": "dual_ridge",
    "elastic-net": "elastic_net_primal",
    "logistic": "logistic_primal",
    "squared-hinge": "squared_hinge_primal",
    "hinge": "hinge_primal",
}
CLASSIFIERS = ("dual_l2_logistic", "dual_l2_svm", "logistic_primal", "squared_hinge_primal",
               "hinge_primal")

_DEFAULTS = dict(objective="dual-logistic", lam=1.0, devices=1, t2=1, epochs=2, threads=1,
                 seed=0, max_rounds=20, target_gap=None, l1_ratio=1.0, smoothing=1.0)


class NotFittedError(ValueError, AttributeError):
    pass


def normalize_labels(y):
    """Binary labels -> +-1 (svmlight.ts:48-63, modelio.py:82-89)."""
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    distinct = np.unique(y)
    bad = distinct[~np.isin(distinct, (-1.0, 0.0, 1.0))]
    if len(bad):
        raise ValueError(f"labels must be binary (+-1 or 0/1), got {bad[0]!r}")
    if -1.0 in distinct and 0.0 in distinct:
        raise ValueError("labels mix -1 and 0 conventions")
    return np.where(y > 0.0, 1.0, -1.0)


def examples_matrix(X, n_features=None):
    """Example-major CSC (columns = examples, rows = features), the parser's
    layout (data.py:190-239), from a scipy.sparse matrix, a dense 2-D array,
    or a list of rows that are dense lists or sorted (index, value) pairs
    (svmlight.ts FeatureMatrix)."""
    try:
        import scipy.sparse as sp
    except ImportError:  # pragma: no cover
        sp = None
    if sp is not None and sp.issparse(X):
        csr = sp.csr_matrix(X)
        csr.sum_duplicates()
        csr.sort_indices()
        n_rows = n_features if n_features is not None else csr.shape[1]
        return SparseColumnMatrix(n_rows, csr.indptr.astype(np.int64),
                                  csr.indices.astype(np.int32), csr.data.astype(np.float64))
    if isinstance(X, np.ndarray) or (len(X) and not _is_pair_row(X[0])):
        dense = np.asarray(X, dtype=np.float64)
        if dense.ndim != 2:
            raise ValueError("X must be 2-D")
        n, d = dense.shape
        nz = dense != 0.0
        indptr = np.concatenate([[0], np.cumsum(nz.sum(axis=1))]).astype(np.int64)
        rows = np.nonzero(nz)[1].astype(np.int32)
        vals = dense[nz]
        return SparseColumnMatrix(n_features if n_features is not None else d, indptr, rows,
                                  vals)
    indptr, rows, vals = [0], [], []
    max_feat = 0
    for i, row in enumerate(X):
        prev = -1
        for j, v in row:
            if j <= prev:
                raise ValueError(f"row {i}: feature indices must be strictly increasing")
            prev = j
            if v != 0.0:
                rows.append(int(j))
                vals.append(float(v))
        max_feat = max(max_feat, prev + 1)
        indptr.append(len(rows))
    return SparseColumnMatrix(n_features if n_features is not None else max_feat,
                              np.asarray(indptr, dtype=np.int64),
                              np.asarray(rows, dtype=np.int32), np.asarray(vals, dtype=np.float64))


def _is_pair_row(row):
    return len(row) > 0 and isinstance(row[0], (tuple, list))


class GlmEstimator:
    """Local (single-node) estimator over the B200 engine (snap-ml-local).

    Parameters mirror EstimatorParams (estimator.ts:20-40): objective, lam
    (lambda), devices (L), t2, epochs, threads (threads per device: 1 runs the
    deterministic sequential kernel, > 1 the asynchronous TPA-SCD kernel),
    seed, max_rounds, target_gap; l1_ratio for elastic-net; smoothing (mu) for
    the smoothed hinge-loss SVM (objective "hinge").
    """

    def __init__(self, **params):
        unknown = set(params) - set(_DEFAULTS)
        if unknown:
            raise TypeError(f"unknown parameters {sorted(unknown)}")
        self._params = dict(_DEFAULTS, **params)
        self._check_params()
        self._model = None
        self.trace_ = []
        self.n_features_in_ = 0

    # -- params (sklearn conventions; getParams/setParams in estimator.ts) -----
    def get_params(self, deep=True):
        return dict(self._params)

    def set_params(self, **params):
        unknown = set(params) - set(_DEFAULTS)
        if unknown:
            raise ValueError(f"unknown parameters {sorted(unknown)}")
        new = dict(self._params, **params)
        self._check_params(new)
        self._params = new
        return self

    def _check_params(self, p=None):
        p = self._params if p is None else p
        if p["objective"] not in OBJECTIVE_NAMES:
            raise ValueError(f"objective must be one of {sorted(OBJECTIVE_NAMES)}")
        if not p["lam"] > 0:
            raise ValueError("lam must be positive")

    @property
    def kind(self):
        return OBJECTIVE_NAMES[self._params["objective"]]

    @property
    def is_classifier(self):
        return self.kind in CLASSIFIERS

    @property
    def fitted(self):
        return self._model is not None

    # -- training ---------------------------------------------------------------
    def fit(self, X, y):
        """Train with K = 1 node and L = devices (estimator.ts:88-117)."""
        ex = examples_matrix(X)
        y = np.asarray(y, dtype=np.float64).reshape(-1)
        if ex.n_cols == 0:
            raise ValueError("cannot fit on an empty dataset")
        if len(y) != ex.n_cols:
            raise ValueError(f"X has {ex.n_cols} rows but y has {len(y)} labels")
        p = self._params
        kind = self.kind
        if kind in CLASSIFIERS:
            y = normalize_labels(y)
            if len(np.unique(y)) > 2:
                raise ValueError("expected binary labels")
        if kind.startswith("dual_"):
            matrix = ex.scale_columns(y) if kind != "dual_ridge" else ex
            spec = ObjectiveSpec(kind, p["lam"], matrix.n_cols, matrix.n_rows,
                                 target=y if kind == "dual_ridge" else None)
        else:
            matrix = ex.transpose()
            spec = ObjectiveSpec(kind, p["lam"], matrix.n_rows, matrix.n_cols, target=y,
                                 l1_ratio=p["l1_ratio"], smoothing=p["smoothing"])
        cfg = HierarchyConfig(nodes=1, devices=p["devices"], t1=p["max_rounds"], t2=p["t2"],
                              epochs=p["epochs"], threads_per_device=p["threads"],
                              seed=p["seed"])
        eng = Engine(matrix, spec, cfg)
        res = eng.train(StoppingCriteria(max_rounds=p["max_rounds"],
                                         target_gap=p["target_gap"]))
        self._spec = spec
        self._model = {"kind": kind, "lam": float(p["lam"]), "alpha": res.model.alpha,
                       "v": np.asarray(res.v, dtype=np.float64)}
        self.n_features_in_ = ex.n_rows
        self.trace_ = [{"round": r.round, "wall_s": r.wall_s, "sim_cost": r.sim_cost,
                        "objective": r.objective, "gap": r.gap} for r in res.trace.rows]
        self.result_ = res
        return self

    # -- model ------------------------------------------------------------------
    def _require(self):
        if self._model is None:
            raise NotFittedError("estimator is not fitted; call fit() first")
        return self._model

    def coefficients(self):
        """Feature weights w: v / lambda for dual kinds, alpha for primal
        (estimator.ts:79-86, modelio.py:57-61)."""
        return np.asarray(modelio.primal_weights(self._require()), dtype=np.float64)

    coef_ = property(coefficients)

    def objective(self):
        """Final objective F(alpha) of the last fit (the trace's last row)."""
        self._require()
        return float(self.trace_[-1]["objective"])

    def duality_gap(self):
        self._require()
        return self.trace_[-1]["gap"]

    def save(self, path):
        m = self._require()
        modelio.save_model(path, self._spec, m["alpha"], m["v"])

    @classmethod
    def load(cls, path, **params):
        m = modelio.load_model(path)
        name = {v: k for k, v in OBJECTIVE_NAMES.items()}[m["kind"]]
        est = cls(**dict(params, objective=name, lam=float(m["lam"])))
        est._model = m
        est.n_features_in_ = len(modelio.primal_weights(m))
        return est

    # -- prediction ---------------------------------------------------------------
    def _examples(self, X):
        ex = examples_matrix(X)
        if ex.n_rows > self.n_features_in_:
            raise ValueError(f"test data has {ex.n_rows} features, model was fitted with "
                             f"{self.n_features_in_}")
        return ex

    def decision_function(self, X):
        """Scores x^T w on the device (decision_scores, modelio.py:64-75)."""
        self._require()
        ex = self._examples(X)
        if ex.n_cols == 0:
            return np.empty(0)
        return modelio.decision_scores(ex, self.coefficients())

    def predict_proba(self, X):
        """P(y = +1 | x) = 0.5 (1 + tanh(z / 2)) (estimator.ts:119-134)."""
        if not self.is_classifier:
            raise ValueError("predict_proba needs a classification objective")
        return modelio.sigmoid(self.decision_function(X))

    def predict(self, X):
        """Labels in {-1, +1} (+1 iff p >= 0.5) for classifiers, scores for
        regression kinds (estimator.ts:136-139, cli.py:280-289)."""
        if self.is_classifier:
            return np.where(self.predict_proba(X) >= 0.5, 1.0, -1.0)
        return self.decision_function(X)

    def score(self, X, y):
        """Accuracy for classifiers, negative mean squared error otherwise."""
        if self.is_classifier:
            y01 = np.where(normalize_labels(y) > 0, 1.0, 0.0)
            return modelio.accuracy(self.predict_proba(X), y01)
        return -modelio.mean_squared_error(self.decision_function(X), y)

    def evaluate(self, X, y):
        """{"logloss", "accuracy"} or {"mse"} (the CLI's eval, cli.py:290-296),
        computed by the fused prediction kernel."""
        self._require()
        ex = self._examples(X)
        return modelio.evaluate(ex, self.coefficients(), np.asarray(y, dtype=np.float64),
                                classify=self.is_classifier)
