"""Per-device subproblem solver: TPA-SCD on the B200.

Mirrors the reference's solver.py (names, fields, exceptions, semantics) with
the compute in csrc/scd.cu + csrc/prng.cu:

    G(delta) = const + lin . (B delta) + (quad/2) ||B delta||^2 + sum_i g_i(base_i + delta_i)

* `damped_solve(sub, gen, t_epochs, n_threads=1, damping=None)` — solver.py:250-305.
  n_threads == 1 runs the deterministic fixed-permutation kernel (the
  reference's sequential run_pass); n_threads > 1 runs the asynchronous
  TPA-SCD kernel (the reference's lock-free worker threads, solver.py:213-239).
* `PermutationGenerator` keeps the reference's host-visible `state`; keys and
  permutations are produced on the device and the state is advanced by the
  GF(2) jump-ahead (bit-exact with solver.py:64-89).
* `gpu_chunk_runner()` is the drop-in for the reference Engine's device-solve
  hook `chunk_runner(sub, dev, cfg)` (engine.py:177-179, 228-233): it runs the
  subtask through the host-buffer C-ABI `glm_device_solve`.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

_MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
DAMPING_FLOOR = 2.0 ** -20   # solver.py:28
PLATEAU_REL = 1e-12          # solver.py:247


class SolverError(RuntimeError):
    pass


class SolverDivergence(SolverError):
    def __init__(self, msg, diagnostics=None):
        super().__init__(msg)
        self.diagnostics = diagnostics or {}


def _D():
    from . import _device
    return _device


def xorshift64_step(state):
    """One xorshift64(13,7,17) step (solver.py:41-46)."""
    return int(L.lib().glm_xorshift_jump(int(state) & _MASK64, 1))


def splitmix64(x):
    """solver.py:49-54."""
    x = (x + GOLDEN) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def derive_seed(base, *indices):
    """solver.py:57-61."""
    s = splitmix64(base & _MASK64)
    for ix in indices:
        s = splitmix64(s ^ ((ix + 0x632BE59BD9B4E019) & _MASK64))
    return s or GOLDEN


class PermutationGenerator:
    """Deterministic permutation stream (solver.py:64-89), generated on the GPU."""

    def __init__(self, seed):
        self.state = (int(seed) & _MASK64) or GOLDEN

    def next_u64(self):
        self.state = xorshift64_step(self.state)
        return self.state

    def advance(self, steps):
        self.state = int(L.lib().glm_xorshift_jump(self.state, int(steps)))

    def keys_device(self, n):
        D = _D()
        out = torch.empty(max(n, 1), dtype=torch.uint32, device=D.device())
        if n > 0:
            L.check(L.lib().glm_perm_keys(self.state, n, D.ptr(out), D.sptr()), "glm_perm_keys")
            self.advance(n)
        return out[:n]

    def keys(self, n):
        return _D().to_host(self.keys_device(n)).astype(np.uint32)

    def permute_device(self, n):
        """Stable argsort of the next n keys (int32, on device): the solver's
        fused path (glm_perm, keys regenerated, never stored)."""
        D = _D()
        if n <= 0:
            return torch.empty(0, dtype=torch.int32, device=D.device())
        perm = _fused_perm(L.lib().glm_perm, self.state, n, "glm_perm")
        self.advance(n)
        return perm

    def permute(self, n):
        if n <= 0:
            return np.empty(0, dtype=np.int64)
        return _D().to_host(self.permute_device(n)).astype(np.int64)


def _fused_perm(fn, seed, n, name):
    D = _D()
    perm = torch.empty(n, dtype=torch.int32, device=D.device())
    nb = L.lib().glm_argsort_temp_bytes(n)
    tmp = torch.empty(nb, dtype=torch.uint8, device=D.device())
    L.check(fn(int(seed) & ((1 << 64) - 1), n, D.ptr(perm), D.ptr(tmp), nb, D.sptr()), name)
    return perm


def argsort_u32_device(keys):
    """np.argsort(keys, kind='stable') on the GPU (prng.cu bucket argsort)."""
    D = _D()
    n = int(keys.numel())
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=keys.device)
    if n:
        nb = L.lib().glm_argsort_temp_bytes(n)
        tmp = torch.empty(nb, dtype=torch.uint8, device=keys.device)
        L.check(L.lib().glm_argsort_u32(D.ptr(keys), n, D.ptr(perm), D.ptr(tmp), nb, D.sptr()),
                "glm_argsort_u32")
    return perm[:n]


@dataclass
class DampingState:
    """Step-scaling factor; only powers of two (solver.py:92-104)."""
    delta: float = 1.0
    last_subproblem_value: float = math.nan

    def halve(self):
        self.delta *= 0.5
        return self.delta

    def reset(self):
        self.delta = 1.0
        self.last_subproblem_value = math.nan


@dataclass
class LocalSubproblem:
    """Quadratic-plus-separable model handed to a device solver (solver.py:107-135).
    lin/base may be numpy arrays or CUDA tensors; data a SparseColumnMatrix,
    DenseColumnMatrix or DeviceMatrix."""
    spec: object
    lin: object
    quad: float
    const: float
    base: object
    data: object
    col_ids: np.ndarray

    @property
    def n_local(self):
        return len(self.base)

    def _dm(self):
        return self.data.device() if hasattr(self.data, "device") else self.data

    def value(self, delta):
        """G(delta) with B delta recomputed exactly (SpMV on the GPU)."""
        D = _D()
        dm = self._dm()
        w = dm.matvec(D.to_device(delta))
        return self.value_given_w(delta, w)

    def value_given_w(self, delta, w):
        D = _D()
        lin = D.to_device(self.lin)
        wd = D.to_device(w)
        c = torch.tensor([float(self.const)], dtype=torch.float64, device=lin.device)
        out = torch.empty(1, dtype=torch.float64, device=lin.device)
        # const + lin.w + quad/2 |w|^2 == glm_inner_model(grad=lin, vbar=w, qo=quad, K=L=1)
        lin_scratch = torch.empty_like(lin)
        L.check(L.lib().glm_inner_model(D.ptr(lin), D.ptr(wd), lin.numel(), float(self.quad),
                                        D.ptr(c), 1.0, 1.0, D.ptr(lin_scratch), D.ptr(out),
                                        D.ptr(D.scratch()), D.sptr()), "glm_inner_model")
        t = D.to_device(self.base) + D.to_device(delta)
        y = D.to_device(self.spec.coord_target[self.col_ids]) \
            if self.spec.coord_target is not None else None
        return float(out.item()) + D.gsum(self.spec, t, y)


@dataclass
class SubtaskResult:
    """Device update (solver.py:138-149)."""
    col_ids: np.ndarray
    delta_alpha: object
    delta_v: object
    epochs_run: int
    final_subproblem_value: float
    initial_subproblem_value: float
    epoch_values: list = field(default_factory=list)
    retries: int = 0
    measured_theta: float | None = None


# ------------------------------------------------------------------ solvers
class DeviceSolver:
    """Owns a glm_solver (scratch + device SolveState) for partitions up to
    (max_coords, max_rows)."""

    def __init__(self, max_coords, max_rows, device=None):
        D = _D()
        D.require_cuda()
        self.device = torch.cuda.current_device() if device is None else device
        self.max_coords = int(max_coords)
        self.max_rows = int(max_rows)
        h = ctypes.c_void_p()
        L.check(L.lib().glm_solver_create(self.device, self.max_coords, self.max_rows,
                                          ctypes.byref(h)), "glm_solver_create")
        self.handle = h
        self.epoch_values = np.zeros(256)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                L.lib().glm_solver_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def set_state(self, gen_state, damping, stream=None):
        L.check(L.lib().glm_solver_set_state(self.handle, int(gen_state) & _MASK64,
                                             float(damping), _D().sptr(stream)),
                "glm_solver_set_state")

    def prepare(self, dm, stream=None):
        """Packed per-coordinate records of a CSC partition for the async
        epoch kernel (glm_solver_prepare); a no-op for dense data."""
        L.check(L.lib().glm_solver_prepare(self.handle, ctypes.byref(dm.struct),
                                           _D().sptr(stream)), "glm_solver_prepare")

    def solve(self, dm, spec, *, lin, cnst, base, quad, epochs, mode, delta_out, dv_out,
              coord_target=None, reset_damping=False, max_attempts=0, group_lanes=0,
              max_inflight=0, accumulate=False, flags=0, stream=None, peer=None):
        """Enqueue one subtask; if max_attempts == 0 returns the GlmSolveResult."""
        D = _D()
        a = L.GlmSolveArgs()
        a.kind = spec.index
        a.mode = mode
        a.lam = spec.lam
        a.l1_ratio = getattr(spec, "l1_ratio", 1.0)
        a.quad = float(quad)
        a.cnst = cnst.data_ptr()
        a.lin = lin.data_ptr()
        a.base = base.data_ptr()
        a.coord_target = coord_target.data_ptr() if coord_target is not None else None
        a.epochs = int(epochs)
        a.max_attempts = int(max_attempts)
        a.group_lanes = int(group_lanes)
        a.max_inflight = int(max_inflight)
        a.accumulate = 1 if accumulate else 0
        a.flags = int(flags)
        a.peer = peer.handle if peer is not None else None
        a.reset_damping = 1 if reset_damping else 0
        res = L.GlmSolveResult()
        st = L.lib().glm_solve(self.handle, ctypes.byref(dm.struct), ctypes.byref(a),
                               D.ptr(delta_out), D.ptr(dv_out),
                               ctypes.byref(res) if max_attempts == 0 else None,
                               D.sptr(stream))
        if st == L.GLM_DIVERGENCE:
            raise SolverDivergence(L.last_error(), diagnostics={
                "value": res.final_value, "retries": res.retries, "damping": res.damping})
        L.check(st, "glm_solve")
        return res if max_attempts == 0 else None

    def join(self, stream=None):
        """Make `stream` wait for this solver's pending permutation prefetch."""
        L.check(L.lib().glm_solver_join(self.handle, _D().sptr(stream)), "glm_solver_join")

    def timing(self, enable=True):
        L.check(L.lib().glm_solver_timing(self.handle, 1 if enable else 0), "glm_solver_timing")

    def timing_read(self, consume=True):
        """(perm_ms, epoch_ms, value_ms) summed over attempts, attempts.
        consume=False keeps graph-captured events for the next replay."""
        ms = np.zeros(3)
        n = np.zeros(1, dtype=np.int32)
        fn = L.lib().glm_solver_timing_read if consume else L.lib().glm_solver_timing_peek
        L.check(fn(self.handle, ms.ctypes.data_as(ctypes.c_void_p),
                   n.ctypes.data_as(ctypes.c_void_p)), "glm_solver_timing_read")
        return ms, int(n[0])

    def timing_glue(self, consume=True):
        """(finalize_ms, round_start_ms, turn_ms) summed, and their counts."""
        ms = np.zeros(3)
        n = np.zeros(3, dtype=np.int32)
        L.check(L.lib().glm_solver_timing_glue(self.handle, ms.ctypes.data_as(ctypes.c_void_p),
                                               n.ctypes.data_as(ctypes.c_void_p),
                                               1 if consume else 0), "glm_solver_timing_glue")
        return ms, n

    def result(self, stream=None):
        res = L.GlmSolveResult()
        ev = self.epoch_values
        L.check(L.lib().glm_solver_result(self.handle, ctypes.byref(res),
                                          ev.ctypes.data_as(ctypes.c_void_p), len(ev),
                                          _D().sptr(stream)), "glm_solver_result")
        return res, ev[:min(res.epochs_run, len(ev))].tolist()


_pool = {}
_pool_lock = threading.Lock()


def _pooled_solver(m, d):
    key = torch.cuda.current_device()
    with _pool_lock:
        s = _pool.get(key)
        if s is None or s.max_coords < m or s.max_rows < d:
            s = DeviceSolver(max(m, 1), max(d, 1))
            _pool[key] = s
        return s


def mode_for_threads(n_threads):
    return L.MODE_SEQUENTIAL if n_threads <= 1 else L.MODE_ASYNC


def damped_solve(sub, gen, t_epochs, n_threads=1, damping=None, mode=None):
    """Run up to t_epochs SCD passes, discarding any pass that increases G
    (solver.py:250-305) — on the GPU. Returns arrays of the same kind as
    sub.base (numpy in, numpy out; CUDA tensor in, CUDA tensor out)."""
    if t_epochs < 1:
        raise ValueError("t_epochs must be >= 1")
    D = _D()
    state = damping if damping is not None else DampingState()
    dm = sub.data.device() if hasattr(sub.data, "device") else sub.data
    m, d = dm.n_cols, dm.n_rows
    host_out = not isinstance(sub.base, torch.Tensor)
    lin = D.to_device(sub.lin)
    base = D.to_device(sub.base)
    y = None
    if sub.spec.coord_target is not None:
        y = D.to_device(np.asarray(sub.spec.coord_target)[np.asarray(sub.col_ids)])
    cnst = torch.tensor([float(sub.const)], dtype=torch.float64, device=lin.device)
    solver = _pooled_solver(m, d)
    solver.set_state(gen.state, state.delta)
    delta = torch.empty(max(m, 1), dtype=torch.float64, device=lin.device)
    dv = torch.empty(max(d, 1), dtype=torch.float64, device=lin.device)
    md = mode if mode is not None else mode_for_threads(n_threads)
    try:
        solver.solve(dm, sub.spec, lin=lin, cnst=cnst, base=base, quad=sub.quad,
                     epochs=t_epochs, mode=md, delta_out=delta, dv_out=dv, coord_target=y)
    finally:
        res, values = solver.result()
        gen.state = int(res.gen_state)
        state.delta = float(res.damping)
    state.last_subproblem_value = float(res.final_value)
    delta, dv = delta[:m], dv[:d]
    if host_out:
        delta, dv = D.to_host(delta).copy(), D.to_host(dv).copy()
    return SubtaskResult(col_ids=sub.col_ids, delta_alpha=delta, delta_v=dv,
                         epochs_run=int(res.epochs_run),
                         final_subproblem_value=float(res.final_value),
                         initial_subproblem_value=float(res.initial_value),
                         epoch_values=values, retries=int(res.retries))


def coordinate_update(spec, rows, vals, sqnorm, t_cur, view, quad):
    """Undamped 1-D step for one coordinate (solver.py:152-187), GPU kernels."""
    D = _D()
    rows = np.asarray(rows, dtype=np.int32)
    vals = np.asarray(vals, dtype=np.float64)
    view = np.asarray(view, dtype=np.float64)
    from .data import DeviceMatrix
    dm = DeviceMatrix.from_csc(len(view), np.array([0, len(rows)], np.int64), rows, vals)
    ga = dm.rmatvec(view) if len(rows) else torch.zeros(1, dtype=torch.float64,
                                                        device=D.device())
    c = torch.tensor([quad * sqnorm], dtype=torch.float64, device=ga.device)
    t = torch.tensor([t_cur], dtype=torch.float64, device=ga.device)
    step = torch.empty(1, dtype=torch.float64, device=ga.device)
    st = L.lib().glm_coordinate_steps(spec.index, spec.lam, getattr(spec, "l1_ratio", 1.0), None,
                                      D.ptr(ga), D.ptr(c), D.ptr(t), 1, D.ptr(step), D.sptr())
    if st == L.GLM_SOLVER_ERROR:
        raise SolverError("non-finite coordinate update")
    L.check(st, "glm_coordinate_steps")
    return float(step.item())


# --------------------------------------------------- reference-engine hook
class _CtxCache:
    """One device context per matrix.  The reference calls the hook from one
    thread per device (engine.py:259-263): creation is locked, and calls on
    one context are serialised by its own lock (calls on different contexts
    run concurrently; ctypes releases the GIL)."""

    def __init__(self):
        self.ctx = {}
        self.lock = threading.Lock()
        self.call_locks = {}

    def call_lock(self, data):
        with self.lock:
            return self.call_locks.setdefault(id(data), threading.Lock())

    def get(self, data):
        with self.lock:
            return self._get(data)

    def _get(self, data):
        key = id(data)
        hit = self.ctx.get(key)
        if hit is not None and hit[0] is data:
            return hit[1]
        h = ctypes.c_void_p()
        dev = torch.cuda.current_device() if torch.cuda.is_available() else 0
        dense = not hasattr(data, "indptr")
        if dense:
            vals = np.ascontiguousarray(np.asarray(data.to_dense(), dtype=np.float64).T)
            st = L.lib().glm_ctx_create(dev, L.DENSE, data.n_rows, data.n_cols, None, None,
                                        vals.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h))
        else:
            ip = np.ascontiguousarray(data.indptr, dtype=np.int64)
            rw = np.ascontiguousarray(data.rows, dtype=np.int32)
            vl = np.ascontiguousarray(data.vals, dtype=np.float64)
            st = L.lib().glm_ctx_create(dev, L.CSC, data.n_rows, data.n_cols,
                                        ip.ctypes.data_as(ctypes.c_void_p),
                                        rw.ctypes.data_as(ctypes.c_void_p),
                                        vl.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h))
        L.check(st, "glm_ctx_create")
        self.ctx[key] = (data, h)
        return h

    def close(self):
        for _, h in self.ctx.values():
            L.lib().glm_ctx_destroy(h)
        self.ctx.clear()


_KIND_INDEX = {"dual_l2_logistic": 0, "dual_l2_svm": 1, "ridge_primal": 2, "lasso_primal": 3,
               "dual_ridge": 4, "elastic_net_primal": 5, "logistic_primal": 6,
               "squared_hinge_primal": 7, "hinge_primal": 8}


def device_solve_host(ctx, sub, gen_state, damping, epochs, mode, out=None):
    """One glm_device_solve call with host (numpy) buffers; `out` may supply
    (delta, dv) host buffers (e.g. pinned). Returns
    (delta, dv, values, info, scal, gen_state, damping, status)."""
    spec = sub.spec
    m, d = len(sub.base), len(sub.lin)
    lin = np.ascontiguousarray(sub.lin, dtype=np.float64)
    base = np.ascontiguousarray(sub.base, dtype=np.float64)
    y = getattr(spec, "coord_target", None)
    yv = None if y is None else np.ascontiguousarray(np.asarray(y)[np.asarray(sub.col_ids)])
    delta, dv = out if out is not None else (np.empty(max(m, 1)), np.empty(max(d, 1)))
    values = np.empty(max(epochs, 1))
    info = np.zeros(5, dtype=np.int32)
    scal = np.zeros(2)
    gs = ctypes.c_uint64(int(gen_state) & _MASK64)
    dmp = ctypes.c_double(float(damping))
    vp = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = L.lib().glm_device_solve(ctx, _KIND_INDEX[spec.kind], float(spec.lam),
                                  float(getattr(spec, "l1_ratio", 1.0)), vp(yv), vp(lin),
                                  float(sub.quad), float(sub.const), vp(base), ctypes.byref(gs),
                                  ctypes.byref(dmp), int(epochs), int(mode), vp(delta), vp(dv),
                                  vp(values), vp(info), vp(scal))
    return delta[:m], dv[:d], values[:info[0]], info, scal, gs.value, dmp.value, st


def gpu_chunk_runner(mode=None, epochs=None):
    """Drop-in for the reference Engine's `chunk_runner` hook
    (engine.py:177-179, 228-233): `Engine(matrix, spec, cfg,
    chunk_runner=gpu_chunk_runner())` runs every device subtask on the B200
    through glm_device_solve. Semantics of damped_solve(sub, dev.gen,
    cfg.epochs, cfg.threads_per_device, dev.damping); dev.gen.state and
    dev.damping are advanced exactly like the reference's."""
    cache = _CtxCache()

    def runner(sub, dev, cfg):
        ep = cfg.epochs if epochs is None else epochs
        md = mode if mode is not None else mode_for_threads(cfg.threads_per_device)
        ctx = cache.get(sub.data)
        with cache.call_lock(sub.data):
            delta, dv, values, info, scal, gs, dmp, st = device_solve_host(
                ctx, sub, dev.gen.state, dev.damping.delta, ep, md)
        dev.gen.state = gs
        dev.damping.delta = dmp
        if st != L.GLM_OK:
            err = _reference_exceptions(sub)
            if st == L.GLM_DIVERGENCE:
                raise err[1]("damping floor reached without subproblem decrease",
                             diagnostics={"value": scal[1], "retries": int(info[1])})
            if st == L.GLM_SOLVER_ERROR:
                raise err[0](L.last_error())
            L.check(st, "glm_device_solve")
        dev.damping.last_subproblem_value = float(scal[1])
        return SubtaskResult(col_ids=sub.col_ids, delta_alpha=delta.copy(), delta_v=dv.copy(),
                             epochs_run=int(info[0]), final_subproblem_value=float(scal[1]),
                             initial_subproblem_value=float(scal[0]),
                             epoch_values=values.tolist(), retries=int(info[1]))

    runner.close = cache.close
    return runner


def _reference_exceptions(sub):
    """Raise the caller's own SolverError types when driven by the reference
    engine (its module defines them); ours otherwise."""
    import sys
    mod = sys.modules.get(type(sub).__module__)
    se = getattr(mod, "SolverError", SolverError)
    sd = getattr(mod, "SolverDivergence", SolverDivergence)
    return se, sd
