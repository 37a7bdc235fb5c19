"""ctypes wrapper over glm_oracle.c plus the numpy engine glue (TEST INFRASTRUCTURE).

Reference paths are relative to /root/reference/pkg/src/hierglm/.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

__all__ = [
    "KINDS", "kind_index", "OMatrix", "load_lib", "derive_seed", "xorshift64_step",
    "splitmix64", "perm_keys", "permute", "generate_keys", "argsort_stable",
    "coordinate_update", "damped_solve", "chunked_epoch", "matvec", "rmatvec",
    "col_sqnorms", "f_eval", "f_grad", "f_conj", "g_sum", "g_conj_sum", "duality_gap",
    "primal_objective", "partition_bounds", "transpose", "select_columns",
    "scale_columns", "train", "train_chunked", "sigmoid", "log_loss", "accuracy",
    "decision_scores", "beta_of", "init_alpha",
]

KINDS = ("dual_l2_logistic", "dual_l2_svm", "ridge_primal", "lasso_primal",
         "dual_ridge", "elastic_net_primal", "logistic_primal", "squared_hinge_primal",
         "hinge_primal")   # 8: smoothed hinge, target[r] = y_r / mu (glm_oracle.c)
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_LOCK = threading.Lock()

_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_P = ctypes.c_void_p


def kind_index(kind):
    return KINDS.index(kind) if isinstance(kind, str) else int(kind)


def load_lib():
    """Load (building on first use when gcc is available) liboracle.so."""
    global _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "glm_oracle.c")
        if not os.path.exists(path) or (os.path.exists(src) and
                                        os.path.getmtime(src) > os.path.getmtime(path)):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        sig = {
            "or_xorshift64_step": (_u64, [_u64]),
            "or_splitmix64": (_u64, [_u64]),
            "or_derive_seed": (_u64, [_u64, _P, ctypes.c_int]),
            "or_perm_keys": (None, [_P, _i64, _P]),
            "or_stable_argsort_u32": (None, [_P, _i64, _P]),
            "or_permute": (None, [_P, _i64, _P]),
            "or_generate_keys": (None, [_u64, _i64, _P]),
            "or_g_sum": (_dbl, [ctypes.c_int, _dbl, _dbl, _P, _P, _i64]),
            "or_g_conj_sum": (_dbl, [ctypes.c_int, _dbl, _dbl, _P, _P, _i64]),
            "or_f_eval": (_dbl, [ctypes.c_int, _dbl, _P, _P, _i64]),
            "or_f_grad": (None, [ctypes.c_int, _dbl, _P, _P, _i64, _P]),
            "or_f_conj": (_dbl, [ctypes.c_int, _dbl, _P, _P, _i64]),
            "or_matvec": (None, [_i64, _i64, _P, _P, _P, _P, _P]),
            "or_rmatvec": (None, [_i64, _P, _P, _P, _P, _P]),
            "or_col_sqnorms": (None, [_i64, _P, _P, _P]),
            "or_step_from_ga": (ctypes.c_int, [ctypes.c_int, _dbl, _dbl, _dbl, _dbl, _dbl,
                                               _dbl, _P]),
            "or_coordinate_update": (ctypes.c_int, [ctypes.c_int, _dbl, _dbl, _dbl, _P, _P,
                                                    _i64, _dbl, _dbl, _P, _dbl, _P]),
            "or_damped_solve": (ctypes.c_int, [ctypes.c_int, _dbl, _dbl, _P, _i64, _i64, _P,
                                               _P, _P, _P, _dbl, _dbl, _P, _P, ctypes.c_int,
                                               _P, _P, _P, _P, _P]),
            "or_chunked_epoch": (ctypes.c_int, [ctypes.c_int, _dbl, _dbl, _P, _i64, _i64, _P,
                                                _P, _P, _P, _dbl, _dbl, _P, ctypes.c_int, _P,
                                                _u64, _u64, _P, _P, _P, _P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
        return lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class OMatrix:
    """CSC arrays with the reference's dtypes (data.py:51-60)."""
    n_rows: int
    indptr: np.ndarray
    rows: np.ndarray
    vals: np.ndarray
    labels: np.ndarray | None = None

    def __post_init__(self):
        self.n_rows = int(self.n_rows)
        self.indptr = np.ascontiguousarray(self.indptr, dtype=np.int64)
        self.rows = np.ascontiguousarray(self.rows, dtype=np.int32)
        self.vals = np.ascontiguousarray(self.vals, dtype=np.float64)
        if self.labels is not None:
            self.labels = np.ascontiguousarray(self.labels, dtype=np.float64)

    @property
    def n_cols(self):
        return len(self.indptr) - 1

    @property
    def nnz(self):
        return int(self.indptr[-1])

    @classmethod
    def from_npz(cls, z, prefix):
        lab = z[prefix + "labels"] if prefix + "labels" in z else None
        return cls(int(z[prefix + "n_rows"]), z[prefix + "indptr"], z[prefix + "rows"],
                   z[prefix + "vals"], lab)

    def col(self, j):
        lo, hi = self.indptr[j], self.indptr[j + 1]
        return self.rows[lo:hi], self.vals[lo:hi]


# ------------------------------------------------------------------ PRNG
def xorshift64_step(s):
    return int(load_lib().or_xorshift64_step(int(s)))


def splitmix64(x):
    return int(load_lib().or_splitmix64(int(x) & (2 ** 64 - 1)))


def derive_seed(base, *indices):
    idx = np.array([int(i) & (2 ** 64 - 1) for i in indices], dtype=np.uint64)
    return int(load_lib().or_derive_seed(int(base) & (2 ** 64 - 1), _p(idx), len(idx)))


def perm_keys(state, n):
    """PermutationGenerator.keys (solver.py:77-84) -> (keys, new_state)."""
    st = np.array([int(state) or 0x9E3779B97F4A7C15], dtype=np.uint64)
    keys = np.empty(max(n, 0), dtype=np.uint32)
    load_lib().or_perm_keys(_p(st), int(n), _p(keys))
    return keys, int(st[0])


def permute(state, n):
    """PermutationGenerator.permute (solver.py:86-89) -> (perm int64, new_state)."""
    st = np.array([int(state) or 0x9E3779B97F4A7C15], dtype=np.uint64)
    perm = np.empty(max(n, 0), dtype=np.int64)
    if n > 0:
        load_lib().or_permute(_p(st), int(n), _p(perm))
    return perm, int(st[0])


def generate_keys(seed, n):
    """pipeline.generate_keys (pipeline.py:29-73)."""
    keys = np.empty(max(n, 0), dtype=np.uint32)
    if n > 0:
        load_lib().or_generate_keys(int(seed) & (2 ** 64 - 1), int(n), _p(keys))
    return keys


def argsort_stable(keys):
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    perm = np.empty(len(keys), dtype=np.int64)
    if len(keys):
        load_lib().or_stable_argsort_u32(_p(keys), len(keys), _p(perm))
    return perm


# ------------------------------------------------------------ objectives
def beta_of(kind, target=None):
    """ObjectiveSpec.beta (objectives.py:71-73); restated: logistic_primal 1/4,
    smoothed hinge 1/mu (= max |target|, the target carrying y / mu)."""
    k = kind_index(kind)
    if k == 8:
        return float(np.max(np.abs(target)))
    return {0: None, 1: None, 4: None, 6: 0.25}.get(k, 1.0)


def init_alpha(kind, n):
    """ObjectiveSpec.init_alpha (objectives.py:90-94)."""
    return np.full(n, 0.5) if kind_index(kind) == 0 else np.zeros(n)


def _beta(kind, lam, target=None):
    k = kind_index(kind)
    if k in (0, 1, 4):
        return 1.0 / lam
    if k == 8:
        return float(np.max(np.abs(target)))
    return 0.25 if k == 6 else 1.0


def f_eval(kind, lam, target, v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    return float(load_lib().or_f_eval(kind_index(kind), lam, _p(target), _p(v), len(v)))


def f_grad(kind, lam, target, v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty_like(v)
    load_lib().or_f_grad(kind_index(kind), lam, _p(target), _p(v), len(v), _p(out))
    return out


def f_conj(kind, lam, target, w):
    w = np.ascontiguousarray(w, dtype=np.float64)
    return float(load_lib().or_f_conj(kind_index(kind), lam, _p(target), _p(w), len(w)))


def g_sum(kind, lam, alpha, rho=1.0, y=None):
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    return float(load_lib().or_g_sum(kind_index(kind), lam, rho, _p(y), _p(a), len(a)))


def g_conj_sum(kind, lam, s, rho=1.0, y=None):
    s = np.ascontiguousarray(s, dtype=np.float64)
    return float(load_lib().or_g_conj_sum(kind_index(kind), lam, rho, _p(y), _p(s), len(s)))


# ------------------------------------------------------------- matrices
def matvec(m, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(m.n_rows)
    load_lib().or_matvec(m.n_rows, m.n_cols, _p(m.indptr), _p(m.rows), _p(m.vals), _p(x),
                         _p(out))
    return out


def rmatvec(m, w):
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.empty(m.n_cols)
    load_lib().or_rmatvec(m.n_cols, _p(m.indptr), _p(m.rows), _p(m.vals), _p(w), _p(out))
    return out


def col_sqnorms(m):
    out = np.empty(m.n_cols)
    load_lib().or_col_sqnorms(m.n_cols, _p(m.indptr), _p(m.vals), _p(out))
    return out


def duality_gap(kind, lam, m, alpha, v, target=None, rho=1.0, y=None):
    """objectives.duality_gap (objectives.py:223-234)."""
    w = f_grad(kind, lam, target, v)
    s = -rmatvec(m, w)
    return (f_eval(kind, lam, target, v) + f_conj(kind, lam, target, w)
            + g_sum(kind, lam, alpha, rho, y) + g_conj_sum(kind, lam, s, rho, y))


def primal_objective(kind, lam, m, alpha, target=None, rho=1.0, y=None):
    """objectives.primal_objective (objectives.py:200-202)."""
    return f_eval(kind, lam, target, matvec(m, alpha)) + g_sum(kind, lam, alpha, rho, y)


def coordinate_update(kind, lam, rows, vals, sqnorm, t, view, quad, rho=1.0, y=0.0):
    """solver.coordinate_update (solver.py:152-187); raises on solver error."""
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    view = np.ascontiguousarray(view, dtype=np.float64)
    out = np.zeros(1)
    st = load_lib().or_coordinate_update(kind_index(kind), lam, rho, y, _p(rows), _p(vals),
                                         len(rows), sqnorm, t, _p(view), quad, _p(out))
    if st:
        raise RuntimeError(f"oracle coordinate_update status {st}")
    return float(out[0])


def damped_solve(kind, lam, m, lin, quad, const, base, gen_state, epochs, damping=1.0,
                 rho=1.0, y=None):
    """solver.damped_solve (solver.py:250-305), sequential (n_threads=1)."""
    lin = np.ascontiguousarray(lin, dtype=np.float64)
    base = np.ascontiguousarray(base, dtype=np.float64)
    yv = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    st = np.array([int(gen_state) or 0x9E3779B97F4A7C15], dtype=np.uint64)
    delta = np.zeros(m.n_cols)
    dv = np.zeros(m.n_rows)
    values = np.zeros(max(epochs, 1))
    info = np.zeros(3, dtype=np.int32)
    vio = np.array([damping, 0.0, 0.0])
    status = load_lib().or_damped_solve(
        kind_index(kind), lam, rho, _p(yv), m.n_rows, m.n_cols, _p(m.indptr), _p(m.rows),
        _p(m.vals), _p(lin), quad, const, _p(base), _p(st), int(epochs), _p(delta), _p(dv),
        _p(values), _p(info), _p(vio))
    return {"status": int(status), "delta": delta, "dv": dv,
            "values": values[:info[0]].copy(), "epochs_run": int(info[0]),
            "retries": int(info[1]), "plateaued": bool(info[2]), "damping": float(vio[0]),
            "initial": float(vio[1]), "final": float(vio[2]), "gen_state": int(st[0])}


def chunked_epoch(kind, lam, m, lin, quad, const, base, offsets, seed, epoch_index, delta,
                  view, damping, rho=1.0, y=None):
    """pipeline.pipelined_epoch(pipelined=False) (pipeline.py:200-242); in-place."""
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    dmp = np.array([damping])
    val = np.zeros(1)
    yv = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    status = load_lib().or_chunked_epoch(
        kind_index(kind), lam, rho, _p(yv), m.n_rows, m.n_cols, _p(m.indptr), _p(m.rows),
        _p(m.vals), _p(np.ascontiguousarray(lin)), quad, const,
        _p(np.ascontiguousarray(base)), len(offs) - 1, _p(offs), int(seed), int(epoch_index),
        _p(dmp), _p(delta), _p(view), _p(val))
    return int(status), float(val[0]), float(dmp[0])


# ------------------------------------------------------------ data layer
def partition_bounds(n_cols, n_nodes, n_devices, strategy="contiguous", col_nnz=None):
    """partition_columns (data.py:264-304) -> W+1 contiguous bounds."""
    workers = n_nodes * n_devices
    if n_nodes < 1 or n_devices < 1 or n_cols < 1 or workers > n_cols:
        raise ValueError("impossible partition")
    if strategy == "contiguous":   # np.array_split sizes
        q, r = divmod(n_cols, workers)
        sizes = [q + 1] * r + [q] * (workers - r)
        return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    csum = np.cumsum(np.asarray(col_nnz, dtype=np.int64))
    total = csum[-1] if n_cols else 0
    bounds = [0]
    for mm in range(1, workers):
        b = int(np.searchsorted(csum, total * mm / workers))
        b = max(b, bounds[-1] + 1)
        b = min(b, n_cols - (workers - mm))
        bounds.append(b)
    bounds.append(n_cols)
    return np.array(bounds, dtype=np.int64)


def transpose(m):
    """SparseColumnMatrix.transpose (data.py:155-165)."""
    order = np.argsort(m.rows, kind="stable")
    new_cols = m.rows[order]
    col_of = np.repeat(np.arange(m.n_cols, dtype=np.int32), np.diff(m.indptr))
    indptr = np.zeros(m.n_rows + 1, dtype=np.int64)
    np.add.at(indptr[1:], new_cols, 1)
    np.cumsum(indptr, out=indptr)
    return OMatrix(m.n_cols, indptr, col_of[order], m.vals[order])


def select_columns(m, cols):
    """SparseColumnMatrix.select_columns (data.py:132-145)."""
    cols = np.asarray(cols, dtype=np.int64)
    counts = np.diff(m.indptr)[cols]
    indptr = np.zeros(len(cols) + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    take = np.concatenate([np.arange(m.indptr[j], m.indptr[j + 1]) for j in cols]) \
        if len(cols) else np.zeros(0, np.int64)
    take = take.astype(np.int64)
    lab = m.labels[cols] if m.labels is not None else None
    return OMatrix(m.n_rows, indptr, m.rows[take], m.vals[take], lab)


def scale_columns(m, scales):
    """SparseColumnMatrix.scale_columns (data.py:147-153)."""
    scales = np.asarray(scales, dtype=np.float64)
    return OMatrix(m.n_rows, m.indptr.copy(), m.rows.copy(),
                   m.vals * np.repeat(scales, np.diff(m.indptr)),
                   None if m.labels is None else m.labels.copy())


# ------------------------------------------------------------- engine
def train(m, kind, lam, *, target=None, nodes=1, devices=1, t2=1, epochs=1, seed=0,
          rounds=1, sigma=None, sigma_bar=None, strategy="contiguous", rho=1.0, y=None,
          parallel=False, target_gap=None, time_budget_s=None, record_gap=True,
          record_obj=True, target_rel_gap=None):
    """Engine.train (engine.py:169-417) restated: K nodes x L devices, t2 inner rounds.

    Returns dict(objective, gap, alpha, v, rounds). With parallel=True, the
    per-device damped solves of one inner round run on host threads (the C
    solver releases the GIL), like the reference's multi-process CLI mode.
    """
    import time
    k = kind_index(kind)
    K, L = nodes, devices
    sig = float(K if sigma is None else sigma)
    sigb = float(L if sigma_bar is None else sigma_bar)
    beta = _beta(k, lam, target)
    bounds = partition_bounds(m.n_cols, K, L, strategy,
                              np.diff(m.indptr) if strategy != "contiguous" else None)
    subs = []
    gens = []
    for w in range(K * L):
        cols = np.arange(bounds[w], bounds[w + 1])
        subs.append((cols, select_columns(m, cols)))
        node, dev = divmod(w, L)
        gens.append(derive_seed(seed, node * L + dev))    # engine.py:117, 125
    alpha = init_alpha(k, m.n_cols)
    v = matvec(m, alpha)
    objs, gaps = [], []

    def record():
        if not record_obj:
            objs.append(np.nan)
            gaps.append(np.nan)
            return None
        fv = f_eval(k, lam, target, v)
        obj = fv + g_sum(k, lam, alpha, rho, y)
        gap = None
        if record_gap and k != 3 and not (k == 5 and rho >= 1.0):
            gap = duality_gap(k, lam, m, alpha, v, target, rho, y)
        objs.append(obj)
        gaps.append(np.nan if gap is None else gap)
        return gap

    t0 = time.perf_counter()
    gap = record()
    pool = ThreadPoolExecutor(max_workers=K * L) if parallel else None
    done = 0
    round_s = []
    for _ in range(rounds):
        if target_gap is not None and gap is not None and gap <= target_gap:
            break
        # relative target: gap <= rel * |F| of the current round (bench.py's bar)
        if target_rel_gap is not None and gap is not None and \
                gap <= target_rel_gap * abs(objs[-1]):
            break
        tr = time.perf_counter()
        grad = f_grad(k, lam, target, v)                   # engine.py:271
        fv = f_eval(k, lam, target, v)
        qo = sig * beta
        node_results = []
        for node in range(K):
            damp = [1.0] * L                               # engine.py:251-252
            d_sl = [np.zeros(len(subs[node * L + l][0])) for l in range(L)]
            vbar = np.zeros(m.n_rows)
            for _ in range(t2):
                fbar = fv / K + float(np.dot(grad, vbar)) + 0.5 * qo * float(np.dot(vbar, vbar))
                lin = grad + qo * vbar                     # engine.py:156-166
                jobs = []
                for l in range(L):
                    w = node * L + l
                    cols, sm = subs[w]
                    yy = None if y is None else y[cols]
                    base = alpha[cols] + d_sl[l]
                    args = (k, lam, sm, lin, sigb * qo, fbar / L, base, gens[w], epochs,
                            damp[l], rho, yy)
                    jobs.append(pool.submit(damped_solve, *args) if pool else args)
                res = [j.result() if pool else damped_solve(*j) for j in jobs]
                for l, r in enumerate(res):
                    if r["status"]:
                        raise RuntimeError(f"oracle solve status {r['status']}")
                    gens[node * L + l] = r["gen_state"]
                    damp[l] = r["damping"]
                    d_sl[l] += r["delta"]                  # engine.py:264-266
                    vbar += r["dv"]
            node_results.append((d_sl, vbar))
        total = node_results[0][1].copy()                  # canonical_sum (comm.py:41-46)
        for _, vb in node_results[1:]:
            total += vb
        for node, (d_sl, _) in enumerate(node_results):
            for l in range(L):
                alpha[subs[node * L + l][0]] += d_sl[l]
        v += total
        done += 1
        round_s.append(time.perf_counter() - tr)
        gap = record()
        if time_budget_s is not None and time.perf_counter() - t0 > time_budget_s:
            break
    if pool:
        pool.shutdown()
    return {"objective": np.array(objs), "gap": np.array(gaps), "alpha": alpha, "v": v,
            "rounds": done, "round_s": round_s, "wall_s": time.perf_counter() - t0}


def train_chunked(m, kind, lam, chunk_size, *, target=None, epochs=1, seed=0, rounds=1,
                  rho=1.0, y=None):
    """Engine with chunked_device_runner (pipeline.py:298-340), single device."""
    k = kind_index(kind)
    n = m.n_cols
    offsets = np.concatenate([np.arange(0, n, chunk_size), [n]]).astype(np.int64)
    alpha = init_alpha(k, n)
    v = matvec(m, alpha)
    beta = _beta(k, lam, target)
    objs = [f_eval(k, lam, target, v) + g_sum(k, lam, alpha, rho, y)]
    epoch_counter = 0
    for _ in range(rounds):
        grad = f_grad(k, lam, target, v)
        fv = f_eval(k, lam, target, v)
        damping = 1.0
        delta = np.zeros(n)
        view = grad.copy()
        for _ in range(epochs):
            st, val, damping = chunked_epoch(k, lam, m, grad, beta, fv, alpha.copy(), offsets,
                                             seed, epoch_counter, delta, view, damping, rho, y)
            epoch_counter += 1
            if st:
                raise RuntimeError(f"oracle chunked status {st}")
        alpha += delta
        v += matvec(m, delta)
        objs.append(f_eval(k, lam, target, v) + g_sum(k, lam, alpha, rho, y))
    return {"objective": np.array(objs), "alpha": alpha, "v": v}


# ----------------------------------------------------------- prediction
def sigmoid(z):
    """modelio.sigmoid (modelio.py:78-79)."""
    return 0.5 * (1.0 + np.tanh(0.5 * np.asarray(z, dtype=np.float64)))


def log_loss(prob, y01):
    """modelio.log_loss (modelio.py:92-95)."""
    p = np.clip(prob, 1e-15, 1.0 - 1e-15)
    return float(-np.mean(y01 * np.log(p) + (1.0 - y01) * np.log(1.0 - p)))


def accuracy(prob, y01):
    return float(np.mean((prob >= 0.5) == (y01 > 0.5)))


def decision_scores(example_matrix, w):
    """modelio.decision_scores (modelio.py:64-75)."""
    return rmatvec(example_matrix, np.asarray(w)[:example_matrix.n_rows])


_ = math  # keep import for restated helpers
