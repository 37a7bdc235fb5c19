"""Training objectives F(alpha) = f(A alpha) + sum_i g_i(alpha_i).

Mirrors the reference's objectives.py (ObjectiveSpec, objectives.py:39-112)
with the same names, constants and error behaviour. The arithmetic
(f, f', f*, g, g*, duality gap) runs in the fused CUDA kernels of
csrc/objective.cu; the functions here are host entry points that take numpy
or device arrays.

Kinds 0..3 are the reference's (objectives.py:22). Kinds 4..8 are restated
kinds the north star names but the reference does not implement (parity
unpinned):

  dual_ridge            f(v) = ||v||^2/(2 lam), g_i(a) = a^2/2 - y_i a (columns x_i)
  elastic_net_primal    f(v) = ||v - b||^2/2,   g_i(a) = lam (rho|a| + (1-rho) a^2/2)
  logistic_primal       f(v) = sum softplus(-y v), g_i(a) = lam a^2/2, beta = 1/4
  squared_hinge_primal  f(v) = 1/2 sum max(0, 1 - y v)^2, g_i(a) = lam a^2/2
  hinge_primal          f(v) = sum h_mu(y v), g_i(a) = lam a^2/2, beta = 1/mu: the
                        hinge loss smoothed over a width mu = `smoothing`
                        (h_mu(z) = 0 for z >= 1, (1-z)^2/(2 mu) above 1 - mu,
                        1 - z - mu/2 below); mu -> 0 is the hinge-loss SVM.
                        The device kernels read its row target as y / mu.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

KINDS = ("dual_l2_logistic", "dual_l2_svm", "ridge_primal", "lasso_primal",
         "dual_ridge", "elastic_net_primal", "logistic_primal", "squared_hinge_primal",
         "hinge_primal")
REFERENCE_KINDS = KINDS[:4]

BOUNDARY_EPS = 1e-12  # objectives.py:26


class UnsupportedObjectiveError(ValueError):
    pass


@dataclass(frozen=True)
class ObjectiveSpec:
    """Objective selection plus the constants the rate bounds need
    (objectives.py:39-112). `target` is b for primal kinds (length = rows),
    and the per-example label/response y for logistic_primal,
    squared_hinge_primal, hinge_primal and dual_ridge. `l1_ratio` is
    elastic-net rho; `smoothing` is the hinge_primal smoothing width mu."""

    kind: str
    lam: float
    n_examples: int
    n_features: int
    target: np.ndarray | None = None
    l1_ratio: float = 1.0
    smoothing: float = 1.0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise UnsupportedObjectiveError(f"unknown objective kind {self.kind!r}")
        if self.lam <= 0:
            raise ValueError("lambda must be positive")
        if self.kind in ("ridge_primal", "lasso_primal", "elastic_net_primal",
                         "logistic_primal", "squared_hinge_primal", "hinge_primal",
                         "dual_ridge") \
                and self.target is None:
            raise ValueError(f"{self.kind} requires a target vector")
        if self.kind == "elastic_net_primal" and not (0.0 <= self.l1_ratio <= 1.0):
            raise ValueError("l1_ratio must lie in [0, 1]")
        if self.kind == "hinge_primal" and not self.smoothing > 0.0:
            raise ValueError("smoothing must be positive")

    @property
    def index(self) -> int:
        return KINDS.index(self.kind)

    @property
    def is_dual(self) -> bool:
        return self.kind.startswith("dual_")

    @property
    def n_coordinates(self):
        """Length of alpha: examples for dual kinds, features for primal."""
        return self.n_examples if self.is_dual else self.n_features

    @property
    def dim(self):
        """Length of the shared vector v = A alpha."""
        return self.n_features if self.is_dual else self.n_examples

    @property
    def beta(self):
        if self.is_dual:
            return 1.0 / self.lam
        if self.kind == "hinge_primal":
            return 1.0 / self.smoothing
        return 0.25 if self.kind == "logistic_primal" else 1.0

    @property
    def mu(self):
        if self.kind == "dual_l2_logistic":
            return 4.0
        if self.kind in ("ridge_primal", "logistic_primal", "squared_hinge_primal",
                         "hinge_primal"):
            return self.lam
        if self.kind == "dual_ridge":
            return 1.0
        if self.kind == "elastic_net_primal":
            return self.lam * (1.0 - self.l1_ratio)
        return 0.0

    @property
    def support_radius(self):
        if self.kind == "dual_l2_svm":
            return math.sqrt(self.n_coordinates)
        return math.inf

    @property
    def has_gap(self) -> bool:
        return not (self.kind == "lasso_primal"
                    or (self.kind == "elastic_net_primal" and self.l1_ratio >= 1.0))

    @property
    def row_target(self):
        """Vector indexed by rows of A (b or y per example) or None; for
        hinge_primal y / mu (the kernels take the label from its sign and the
        smoothing width from its magnitude)."""
        if self.is_dual or self.target is None:
            return None
        if self.kind == "hinge_primal":
            return np.asarray(self.target, dtype=np.float64) / self.smoothing
        return self.target

    @property
    def coord_target(self):
        """Vector indexed by coordinates (dual_ridge y) or None."""
        return self.target if self.kind == "dual_ridge" else None

    def init_alpha(self):
        n = self.n_coordinates
        if self.kind == "dual_l2_logistic":
            return np.full(n, 0.5)
        return np.zeros(n)

    def domain(self):
        if self.kind == "dual_l2_logistic":
            return (BOUNDARY_EPS, 1.0 - BOUNDARY_EPS)
        if self.kind == "dual_l2_svm":
            return (0.0, 1.0)
        return (-math.inf, math.inf)

    def check_alpha(self, alpha):
        alpha = np.asarray(alpha)
        if not np.all(np.isfinite(alpha)):
            raise ValueError("alpha contains non-finite entries")
        if self.kind == "dual_l2_logistic":
            if np.any(alpha <= 0.0) or np.any(alpha >= 1.0):
                raise ValueError("dual logistic alpha must stay inside (0, 1)")
        elif self.kind == "dual_l2_svm":
            if np.any(alpha < 0.0) or np.any(alpha > 1.0):
                raise ValueError("dual svm alpha must stay inside [0, 1]")


@dataclass
class Model:
    alpha: np.ndarray
    spec: ObjectiveSpec


@dataclass
class SharedVector:
    v: np.ndarray
    stamp: int = 0


def _dev():
    from . import _device
    return _device


def f_eval(spec, v):
    """f(v) (objectives.py:129-133), computed on the GPU."""
    D = _dev()
    vd = D.to_device(v)
    tgt = D.to_device(spec.row_target) if spec.row_target is not None else None
    return float(D.fgrad(spec, vd, tgt, want_grad=False)[1])


def f_grad(spec, v):
    """f'(v) (objectives.py:136-139) as a numpy array (GPU kernel)."""
    D = _dev()
    vd = D.to_device(v)
    tgt = D.to_device(spec.row_target) if spec.row_target is not None else None
    return D.to_host(D.fgrad(spec, vd, tgt, want_grad=True)[0])


def g_sum(spec, alpha):
    """sum_i g_i(alpha_i) (objectives.py:165-173), GPU reduction."""
    D = _dev()
    y = D.to_device(spec.coord_target) if spec.coord_target is not None else None
    return D.gsum(spec, D.to_device(alpha), y)


def primal_objective(spec, matrix, alpha):
    """F(alpha) = f(A alpha) + sum g (objectives.py:200-202)."""
    dm = matrix.device() if hasattr(matrix, "device") else matrix
    D = _dev()
    a = D.to_device(alpha)
    return f_eval(spec, dm.matvec(a)) + g_sum(spec, a)


def duality_gap(spec, matrix, alpha, v):
    """Fenchel gap (objectives.py:223-234) via the fused gap kernels."""
    if not spec.has_gap:
        raise UnsupportedObjectiveError(
            "duality gap is not available for lasso_primal; use reference_optimum")
    dm = matrix.device() if hasattr(matrix, "device") else matrix
    terms = _dev().gap_terms(spec, dm, alpha, v)
    return float(terms[0] + terms[1] + terms[2])
