"""Two-level CoCoA engine with device-resident state (B200).

Mirrors the reference's engine.py (HierarchyConfig, StoppingCriteria,
ConvergenceTrace, TrainResult, Engine, train; engine.py:34-423) with the same
round semantics:

    lin = grad f(v) + sigma*beta*v_bar,  quad = sigma_bar*sigma*beta
    const = (f(v)/K + grad.v_bar + sigma*beta/2 |v_bar|^2) / L

but alpha, v, grad, lin, v_bar and every per-device delta live in HBM; each
round runs the fused kernels of libglm_b200.so and, across processes, one
NCCL allreduce of Delta v (engine.py:282). Nothing leaves the device inside a
round except the solve status; `record()` reads back 4 scalars (the trace).

Topology: all K x L workers of a process share its GPU (virtual devices, used
for parity with the reference's in-process engine), or — with a reducer and
node_index — one process owns node `node_index` (one GPU per process, NCCL
between processes), or — with device_index and a node_reducer as well — one
process owns the single worker (node_index, device_index): the two-level
scheme across GPUs, K x L ranks, each inner round folding the node's Delta v
over the node's ranks (engine.py:259-266) and each outer round summing the
nodes' v_bar over all ranks (engine.py:282).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .data import DeviceMatrix, partition_bounds
from .objectives import Model, SharedVector
from .solver import (DeviceSolver, SolverError, SubtaskResult, derive_seed,
                     mode_for_threads)


def _D():
    from . import _device
    return _device


@dataclass
class HierarchyConfig:
    """Topology and schedule: K nodes x L devices, t1 outer / t2 inner rounds
    (engine.py:34-58)."""
    nodes: int = 1
    devices: int = 1
    t1: int = 1
    t2: int = 1
    sigma: float | None = None
    sigma_bar: float | None = None
    seed: int = 0
    epochs: int = 1
    threads_per_device: int = 1
    partition_strategy: str = "contiguous"

    def __post_init__(self):
        if min(self.nodes, self.devices, self.t1, self.t2, self.epochs) < 1:
            raise ValueError("nodes, devices, t1, t2 and epochs must be >= 1")

    @property
    def sigma_eff(self):
        return float(self.nodes if self.sigma is None else self.sigma)

    @property
    def sigma_bar_eff(self):
        return float(self.devices if self.sigma_bar is None else self.sigma_bar)


@dataclass
class StoppingCriteria:
    max_rounds: int | None = None
    target_gap: float | None = None
    target_subopt: float | None = None
    f_star: float | None = None
    time_budget_s: float | None = None


@dataclass
class TraceRow:
    round: int
    wall_s: float
    sim_cost: float
    objective: float
    gap: float | None
    theta: float | None


class ConvergenceTrace:
    HEADER = "round,wall_s,sim_cost,objective,gap,theta"

    def __init__(self):
        self.rows: list[TraceRow] = []

    def append(self, row):
        self.rows.append(row)

    def objectives(self):
        return np.array([r.objective for r in self.rows])

    def gaps(self):
        return np.array([np.nan if r.gap is None else r.gap for r in self.rows])

    def write_csv(self, path):
        with open(path, "w") as fh:
            fh.write(self.HEADER + "\n")
            for r in self.rows:
                gap = "" if r.gap is None else repr(float(r.gap))
                theta = "" if r.theta is None else repr(float(r.theta))
                fh.write(f"{r.round},{float(r.wall_s)!r},{float(r.sim_cost)!r},"
                         f"{float(r.objective)!r},{gap},{theta}\n")


@dataclass
class TrainResult:
    model: Model
    trace: ConvergenceTrace
    v: np.ndarray
    rounds: int
    stop_reason: str
    theta_bar_max: float | None = None
    theta_bars: list = field(default_factory=list)


class _GenView:
    """PermutationGenerator-like view of a worker's device-held stream state."""

    def __init__(self, state):
        self.state = state


class _DampView:
    def __init__(self):
        self.delta = 1.0
        self.last_subproblem_value = math.nan

    def reset(self):
        self.delta = 1.0
        self.last_subproblem_value = math.nan


class _Worker:
    """One (node, device) partition: a zero-copy column view + its solver."""

    def __init__(self, engine, node, dev, lo, hi, seed_index):
        self.node, self.device_index = node, dev
        self.lo, self.hi = int(lo), int(hi)
        self.cols = np.arange(lo, hi, dtype=np.int64)
        self.data = engine.dm.columns(lo - engine.col_offset, hi - engine.col_offset)
        self.m = self.hi - self.lo
        d = engine.d
        self.solver = DeviceSolver(self.m, d)
        self.gen = _GenView(derive_seed(engine.config.seed, seed_index))
        self.damping = _DampView()
        self.solver.set_state(self.gen.state, 1.0, engine.stream)
        if engine.mode == L.MODE_ASYNC and self.data.layout == L.CSC and self.m > 0:
            self.solver.prepare(self.data, engine.stream)     # packed coordinate records
        self.gsum_ok = False        # solver's cached g-sum matches alpha[cols]
        self.coord_target = None
        ct = engine.spec.coord_target
        if ct is not None:
            self.coord_target = _D().to_device(np.asarray(ct)[lo:hi])
        self.last = None


class Engine:
    """Drives the two-level scheme with the matrix resident in HBM (engine.py:169-407).

    mode: None -> from config.threads_per_device (1 = deterministic sequential
    kernel, >1 = asynchronous TPA-SCD), or 'sequential' / 'async'.
    sync_solves: False lets async solves enqueue a fixed attempt budget
    (epochs + retry_budget) without a host round-trip per subtask.
    """

    def __init__(self, matrix, spec, config, reducer=None, cost_model=None, node_index=None,
                 measure_theta_bar=False, measure_theta_outer=False, chunk_runner=None,
                 mode=None, sync_solves=True, retry_budget=2, group_lanes=0, max_inflight=0,
                 n_total=None, cache_flags=0, peer_exchange=True, peer_timeout=None,
                 device_index=None, node_reducer=None):
        if measure_theta_bar or measure_theta_outer:
            raise ValueError("theta measurement is the reference's CPU test-mode oracle "
                             "(solver.py:308-391); it is out of scope on the device path")
        D = _D()
        D.require_cuda()
        self.spec = spec
        self.config = config
        self.cost_model = cost_model
        self.chunk_runner = chunk_runner
        self.device = D.device()
        self.stream = torch.cuda.current_stream()
        self.mode = {None: mode_for_threads(config.threads_per_device),
                     "sequential": L.MODE_SEQUENTIAL, "async": L.MODE_ASYNC}[mode]
        # sequential solves run the host retry loop unless the caller explicitly
        # enqueues them (sync_solves=False: a fixed attempt budget per subtask)
        self.sync_solves = sync_solves is not False and (sync_solves or
                                                         self.mode == L.MODE_SEQUENTIAL)
        self.retry_budget = int(retry_budget)
        self.group_lanes = int(group_lanes)
        self.max_inflight = int(max_inflight)
        self.cache_flags = int(cache_flags)
        local_input = isinstance(matrix, DeviceMatrix) and node_index is not None
        if device_index is not None and node_index is None:
            raise ValueError("device_index needs node_index (a rank owns one (node, device))")
        if device_index is not None and config.devices > 1 and node_reducer is None:
            raise ValueError("a rank per device needs the node's reducer (node_reducer)")
        self.device_index = None if device_index is None else int(device_index)
        self.node_reducer = node_reducer
        if local_input and n_total is None:
            raise ValueError("a node-local DeviceMatrix needs n_total (global coordinates)")
        n = int(n_total) if local_input else matrix.n_cols
        self.n = n
        col_nnz = None
        if config.partition_strategy != "contiguous":
            col_nnz = matrix.col_nnz() if hasattr(matrix, "col_nnz") else \
                _D().to_host(matrix.indptr[1:] - matrix.indptr[:-1])
        self.bounds = partition_bounds(n, config.nodes, config.devices,
                                       config.partition_strategy, col_nnz)
        K, L_ = config.nodes, config.devices
        if node_index is None:
            local_nodes = list(range(K))
            self.reducer = None
        else:
            if reducer is None:
                raise ValueError("multi-process mode needs a reducer")
            local_nodes = [int(node_index)]
            self.reducer = reducer
        self.local_nodes = local_nodes
        self.node_index = node_index
        # device matrix: the whole matrix in-process, only the node's columns otherwise
        if self.device_index is not None:      # this rank's worker columns only
            w_lo = node_index * L_ + self.device_index
            lo, hi = int(self.bounds[w_lo]), int(self.bounds[w_lo + 1])
        elif node_index is not None:
            lo, hi = int(self.bounds[node_index * L_]), int(self.bounds[(node_index + 1) * L_])
        if local_input:     # caller uploaded only this rank's columns
            self.dm, self.col_offset = matrix, lo
            if matrix.n_cols != hi - lo:
                raise ValueError("local matrix does not match the rank's partition")
        elif isinstance(matrix, DeviceMatrix):
            self.dm, self.col_offset = matrix, 0
        elif node_index is None:
            self.dm, self.col_offset = matrix.device(), 0
        else:
            sub = matrix.select_columns(np.arange(lo, hi)) if not hasattr(matrix, "dense") \
                else None
            self.dm = sub.device() if sub is not None else \
                DeviceMatrix.from_dense(matrix.dense[:, lo:hi])
            self.col_offset = int(lo)
        self.d = self.dm.n_rows
        f = dict(dtype=torch.float64, device=self.device)
        self.workers = {}
        for k in local_nodes:
            for l in (range(L_) if self.device_index is None else [self.device_index]):
                w = k * L_ + l
                self.workers[(k, l)] = _Worker(self, k, l, self.bounds[w], self.bounds[w + 1],
                                               k * L_ + l)
        self.row_target = D.to_device(spec.row_target) if spec.row_target is not None else None
        self.alpha_dev = D.to_device(spec.init_alpha())
        self.v_dev = self._initial_v()
        self._v0 = self.v_dev.clone()
        self.grad = torch.empty(max(self.d, 1), **f)
        self.lin = torch.empty(max(self.d, 1), **f)
        self.vbar = torch.zeros(max(self.d, 1), **f)
        self.total = torch.zeros(max(self.d, 1), **f)
        self.scal = torch.zeros(8, **f)      # [fv, cnst, ...]
        self.gap_out = torch.zeros(4, **f)
        self.w_scratch = torch.empty(max(self.d, 1), **f)
        self.stamp = 0
        self.theta_bars = []
        self._theta_outer_last = None
        self.last_results = []
        # Fused rounds (one local worker, t2 = 1, enqueued solves): the Delta v
        # exchange runs over NVLink peer memory fused with the next round's start
        # (csrc/peer.cu) instead of an NCCL all-reduce + 3 glue kernels; v then
        # lags one round's Delta v until _flush_v() (before anything reads v).
        self.exchange = None
        self._pending = False
        self._turn_ready = False    # the last glm_round_turn already started the next round
        if (peer_exchange and len(self.workers) == 1 and config.t2 == 1
                and chunk_runner is None and not self.sync_solves):
            from .comm import PeerExchange, ReduceError
            try:       # collective: every rank gets an exchange or none does
                self.exchange = PeerExchange(self.d, local=self.reducer is None,
                                             timeout=peer_timeout)
            except ReduceError:        # no P2P between the ranks' GPUs: NCCL path
                self.exchange = None
            if self.exchange is not None:
                self.exchange.consume(self.stream)

    def close(self):
        """Release the peer exchange (IPC mappings) before the process group
        or the CUDA context goes away."""
        if self.exchange is not None:
            self.exchange.close()
            self.exchange = None

    # -- state -----------------------------------------------------------------
    def _initial_v(self):
        """v0 = A alpha0 (engine.py:211-212), deterministic: gather through the
        transpose when alpha0 != 0 (dual logistic), exact zero otherwise."""
        f = dict(dtype=torch.float64, device=self.device)
        if self.spec.kind != "dual_l2_logistic":
            return torch.zeros(max(self.d, 1), **f)
        a0 = self.alpha_dev[self.col_offset:self.col_offset + self.dm.n_cols]
        if self.dm.layout == L.DENSE:
            v = self.dm.matvec(a0).clone()
        else:
            v = self.dm.transpose().rmatvec(a0).clone()
        if self.reducer is not None:
            v = self.reducer.allreduce_inplace(v)
        out = torch.zeros(max(self.d, 1), **f)
        out[:self.d] = v[:self.d]
        return out

    def reset(self):
        """Back to the initial point (engine.py:211-212): alpha0, v0 = A alpha0,
        fresh permutation streams and damping (no re-upload, no SpMV)."""
        self.alpha_dev.copy_(_D().to_device(self.spec.init_alpha()))
        self.v_dev.copy_(self._v0)
        if self.exchange is not None:            # drop the last round's Delta v
            self.exchange.consume(self.stream)
            self._pending = False
            self._turn_ready = False
        for (k, l), wk in self.workers.items():
            wk.gen.state = derive_seed(self.config.seed, k * self.config.devices + l)
            wk.solver.set_state(wk.gen.state, 1.0, self.stream)
            wk.gsum_ok = False
        self.stamp = 0

    def capture(self, rounds, on_round=None):
        """Record `rounds` outer rounds from the current state as one CUDA graph
        (requires sync_solves=False: no host round-trip inside a round; the
        NCCL all-reduce is captured too). Replay after reset():
        ``g = eng.capture(20); eng.reset(); g.replay()``. The graph's first
        round computes G(0) from scratch, so call this right after reset().
        `on_round(r)` (optional) enqueues extra capture-safe work before the
        first round (r = 0) and after round r = 1..rounds, e.g.
        `gap_terms_async` into a per-round slot."""
        if self.sync_solves or self.chunk_runner is not None:
            raise ValueError("graph capture needs sync_solves=False and the device solver")
        D = _D()
        # captured at the highest priority (kernel nodes keep their stream's
        # priority): the round's kernels win SMs over the permutation prefetch
        side = torch.cuda.Stream(priority=-100)
        side.wait_stream(torch.cuda.current_stream())
        D.scratch(side)                        # allocate outside the capture
        graph = torch.cuda.CUDAGraph()
        prev = self.stream
        try:
            with torch.cuda.graph(graph, stream=side):
                self.stream = torch.cuda.current_stream()
                if on_round is not None:
                    on_round(0)
                for r in range(rounds):
                    self.outer_round()
                    if on_round is not None:
                        on_round(r + 1)
                for wk in self.workers.values():   # rejoin the prefetch branches
                    wk.solver.join(self.stream)
        finally:
            self.stream = prev
        return graph

    @property
    def alpha(self):
        return _D().to_host(self.alpha_dev).copy()

    @alpha.setter
    def alpha(self, value):
        self._turn_ready = False
        self.alpha_dev = _D().to_device(value).clone()
        for wk in self.workers.values():
            wk.gsum_ok = False

    def _flush_v(self):
        """Apply the last fused round's Delta v to v (engine.py:306)."""
        if self._pending:
            L.check(L.lib().glm_round_start(
                self.exchange.handle, None, 0, self.spec.index, self.spec.lam, None,
                _D().ptr(self.v_dev), self.d, None, None, None, None, 1.0, 1.0, 0, None,
                _D().sptr(self.stream)), "glm_round_start")
            self._pending = False

    @property
    def v(self):
        self._flush_v()
        return _D().to_host(self.v_dev[:self.d]).copy()

    @v.setter
    def v(self, value):
        if self.exchange is not None:           # a pending Delta v no longer applies
            self.exchange.consume(self.stream)
            self._pending = False
            self._turn_ready = False
        self.v_dev[:self.d] = _D().to_device(value)

    @property
    def shared(self):
        return SharedVector(self.v, self.stamp)

    # -- one round ---------------------------------------------------------------
    def _solve_worker(self, wk, lin, cnst, first_inner, vbar):
        """One device subtask (engine.py:222-237). The solver folds its result
        in place: alpha[cols] += delta (the base of the next inner round is then
        alpha[cols] itself, engine.py:225) and v_bar += Delta v (engine.py:264-266)."""
        cfg = self.config
        D = _D()
        quad = cfg.sigma_bar_eff * cfg.sigma_eff * self.spec.beta
        a_slice = self.alpha_dev[wk.lo:wk.hi]
        if self.chunk_runner is not None:
            from .solver import LocalSubproblem
            if first_inner:
                wk.damping.reset()
            sub = LocalSubproblem(spec=self.spec, lin=lin, quad=quad, const=cnst,
                                  base=a_slice.clone(), data=wk.data, col_ids=wk.cols)
            res = self.chunk_runner(sub, wk, cfg)
            a_slice += D.to_device(res.delta_alpha)
            if self.spec.kind == "dual_l2_svm":     # keep the fold in the box (scd.cu finalize)
                a_slice.clamp_(0.0, 1.0)
            vbar[:self.d] += D.to_device(res.delta_v)
            wk.last = res
            return
        max_attempts = 0 if self.sync_solves else cfg.epochs + self.retry_budget
        flags = self.cache_flags | L.FLAG_PREFETCH_PERM | (L.FLAG_REUSE_GSUM if wk.gsum_ok
                                                              else 0)
        res = wk.solver.solve(wk.data, self.spec, lin=lin, cnst=cnst, base=a_slice,
                              quad=quad, epochs=cfg.epochs, mode=self.mode,
                              delta_out=a_slice, dv_out=vbar, coord_target=wk.coord_target,
                              reset_damping=first_inner, max_attempts=max_attempts,
                              group_lanes=self.group_lanes, max_inflight=self.max_inflight,
                              accumulate=True, flags=flags, stream=self.stream)
        # alpha[cols] now holds base + delta, whose g-sum the solver cached
        wk.gsum_ok = True
        wk.last = res

    def _run_node(self, k, vbar):
        """t2 inner rounds for node k (engine.py:239-267); accumulates the
        node's v_bar into `vbar` (zeroed by the caller)."""
        cfg = self.config
        D = _D()
        L_ = cfg.devices
        qo = cfg.sigma_eff * self.spec.beta
        per_rank = self.device_index is not None
        wks = [self.workers[(k, l)] for l in
               ([self.device_index] if per_rank else range(L_))]
        for t in range(cfg.t2):
            if t > 0 or not self._lin_fresh:
                # lin = grad + qo*vbar ; cnst = (fv/K + grad.vbar + qo/2|vbar|^2)/L
                # (t == 0 of a later node: v_bar = 0, rebuild what node k-1 overwrote)
                L.check(L.lib().glm_inner_model(
                    D.ptr(self.grad), D.ptr(vbar) if t > 0 else None, self.d, qo,
                    D.ptr(self.scal[0:1]),
                    float(cfg.nodes), float(L_), D.ptr(self.lin), D.ptr(self.scal[1:2]),
                    D.ptr(D.scratch(self.stream)), D.sptr(self.stream)), "glm_inner_model")
            cnst = self.scal[1:2] if self.chunk_runner is None else float(self.scal[1].item())
            # the devices of an inner round read lin/cnst, not v_bar, so folding
            # each result into v_bar as it lands keeps the reference's device-order
            # sum (engine.py:264-266) without a second pass
            self._lin_fresh = False
            if per_rank:
                # this rank's device solves into a zeroed Delta v; the node's
                # ranks then fold every device's Delta v into v_bar in device
                # order — the same additions, in the same order, as the
                # in-process fold below (engine.py:264-266)
                dv = self._dv_local()
                self._solve_worker(wks[0], self.lin, cnst, first_inner=(t == 0), vbar=dv)
                parts = self.node_reducer.allgather(dv) if L_ > 1 else [dv]
                for part in parts:
                    L.check(L.lib().glm_axpby(self.d, 1.0, D.ptr(part), 1.0, D.ptr(vbar),
                                              D.sptr(self.stream)), "glm_axpby")
                continue
            for wk in wks:                       # canonical device order
                self._solve_worker(wk, self.lin, cnst, first_inner=(t == 0), vbar=vbar)
        return vbar

    def _dv_local(self):
        if getattr(self, "_dv_loc", None) is None:
            self._dv_loc = torch.zeros(max(self.d, 1), dtype=torch.float64, device=self.device)
        self._dv_loc.zero_()
        return self._dv_loc

    def _outer_round_fused(self):
        """One round with the exchange over peer memory: glm_round_start applies
        the previous round's Delta v of every rank (canonical rank order), builds
        the model and starts the solver; the solve publishes its Delta v."""
        D = _D()
        cfg = self.config
        wk = next(iter(self.workers.values()))
        reuse = wk.gsum_ok
        # one attempt per round (no retry budget): the round ends in
        # glm_round_turn, which also starts the next round
        turn = self.retry_budget == 0 and cfg.epochs == 1 and wk.m > 0
        if not (turn and self._turn_ready):
            L.check(L.lib().glm_round_start(
                self.exchange.handle, wk.solver.handle, 2 if reuse else 1, self.spec.index,
                self.spec.lam, D.ptr(self.row_target), D.ptr(self.v_dev), self.d,
                D.ptr(self.grad), D.ptr(self.lin), D.ptr(self.scal[0:1]), D.ptr(self.scal[1:2]),
                float(cfg.nodes), float(cfg.devices), int(cfg.epochs),
                D.ptr(D.scratch(self.stream)), D.sptr(self.stream)), "glm_round_start")
            self._pending = False
        quad = cfg.sigma_bar_eff * cfg.sigma_eff * self.spec.beta
        a_slice = self.alpha_dev[wk.lo:wk.hi]
        flags = self.cache_flags | L.FLAG_PREFETCH_PERM | L.FLAG_PEER_FINALIZE | \
            ((L.FLAG_REUSE_GSUM | L.FLAG_SKIP_BEGIN) if reuse or (turn and self._turn_ready)
             else 0) | (L.FLAG_TURN if turn else 0)
        wk.last = wk.solver.solve(
            wk.data, self.spec, lin=self.lin, cnst=self.scal[1:2], base=a_slice, quad=quad,
            epochs=cfg.epochs, mode=self.mode, delta_out=a_slice, dv_out=None,
            coord_target=wk.coord_target, reset_damping=True,
            max_attempts=cfg.epochs + self.retry_budget, group_lanes=self.group_lanes,
            max_inflight=self.max_inflight, accumulate=True, flags=flags, stream=self.stream,
            peer=self.exchange)
        if turn:
            L.check(L.lib().glm_round_turn(
                self.exchange.handle, wk.solver.handle, self.spec.index, self.spec.lam, quad,
                D.ptr(self.scal[1:2]), D.ptr(a_slice), wk.m, D.ptr(self.row_target),
                D.ptr(self.v_dev), self.d, D.ptr(self.grad), D.ptr(self.lin),
                D.ptr(self.scal[0:1]), float(cfg.nodes), float(cfg.devices), int(cfg.epochs),
                D.ptr(D.scratch(self.stream)), D.sptr(self.stream)), "glm_round_turn")
            self._turn_ready = True
            self._pending = False
        else:
            self._pending = True
        wk.gsum_ok = True
        self.last_results = []
        self.stamp += 1

    def outer_round(self):
        """One outer round (engine.py:269-307): grad/f(v) fused with the first
        inner model, per-node t2 inner rounds, Delta v reduce, v += total."""
        if self.exchange is not None:
            return self._outer_round_fused()
        D = _D()
        cfg = self.config
        L.check(L.lib().glm_outer_model(
            self.spec.index, self.spec.lam, D.ptr(self.row_target), D.ptr(self.v_dev), self.d,
            D.ptr(self.grad), D.ptr(self.lin), D.ptr(self.scal[0:1]), D.ptr(self.scal[1:2]),
            float(cfg.nodes), float(cfg.devices), D.ptr(D.scratch(self.stream)),
            D.sptr(self.stream)), "glm_outer_model")
        self._lin_fresh = True      # lin/cnst hold the t = 0 model (v_bar = 0)
        self.last_results = []
        single = self.reducer is None and len(self.local_nodes) == 1
        try:
            if single:
                self.total.zero_()
                self._run_node(self.local_nodes[0], self.total)
            elif self.reducer is None:
                self.total.zero_()
                for k in self.local_nodes:             # canonical node order (comm.py:41-46)
                    self.vbar.zero_()
                    self._run_node(k, self.vbar)
                    L.check(L.lib().glm_axpby(self.d, 1.0, D.ptr(self.vbar), 1.0,
                                              D.ptr(self.total), D.sptr(self.stream)),
                            "glm_axpby")
            else:
                self.total.zero_()
                self._run_node(self.local_nodes[0], self.total)
                if self.device_index:          # one contribution per node (its device 0)
                    self.total.zero_()
                self.reducer.allreduce_inplace(self.total)   # engine.py:282
        except BaseException:
            if self.reducer is not None and hasattr(self.reducer, "abort"):
                self.reducer.abort()
            raise
        L.check(L.lib().glm_axpby(self.d, 1.0, D.ptr(self.total), 1.0, D.ptr(self.v_dev),
                                  D.sptr(self.stream)), "glm_axpby")   # engine.py:306
        self.stamp += 1

    def check_solves(self):
        """Raise the solver error of the last round's subtasks (deferred when
        solves are enqueued without a host round-trip, sync_solves=False)."""
        if self.exchange is not None:
            try:
                self.exchange.check()          # a device-side wait that timed out
            except BaseException:
                if self.reducer is not None and hasattr(self.reducer, "abort"):
                    self.reducer.abort()
                raise
        if self.sync_solves or self.chunk_runner is not None:
            return
        for wk in self.workers.values():
            res, _ = wk.solver.result(self.stream)
            if res.status == L.GLM_DIVERGENCE:
                from .solver import SolverDivergence
                raise SolverDivergence("damping floor reached without subproblem decrease",
                                       diagnostics={"value": res.final_value,
                                                    "retries": res.retries})
            if res.status != L.GLM_OK:
                raise SolverError("non-finite entries in shared view or coordinate update")

    # -- metrics ---------------------------------------------------------------
    def gap_terms_async(self, out):
        """Enqueue the fused gap kernels (+ the cross-rank sum of their partial
        terms) into the 4-double device tensor `out` without a host round trip
        (capture-safe): objective = out[3] + out[1], gap = out[0] + out[1] +
        out[2] (engine.py:325-351)."""
        self._flush_v()
        D = _D()
        a_local = self.alpha_dev[self.col_offset:self.col_offset + self.dm.n_cols]
        ct = self._gap_coord_target()
        L.check(L.lib().glm_gap_terms(
            ctypes.byref(self.dm.struct), self.spec.index, self.spec.lam, self.spec.l1_ratio,
            D.ptr(self.row_target), D.ptr(ct), D.ptr(a_local), D.ptr(self.v_dev),
            D.ptr(self.w_scratch), D.ptr(out), D.ptr(D.scratch(self.stream)),
            D.sptr(self.stream)), "glm_gap_terms")
        if self.reducer is not None:                 # engine.py:339-341
            self.reducer.allreduce_inplace(out[1:3])
        return out

    def _gap_coord_target(self):
        if self.spec.coord_target is None:
            return None
        if getattr(self, "_gap_ct", None) is None:
            self._gap_ct = _D().to_device(np.asarray(self.spec.coord_target)[
                self.col_offset:self.col_offset + self.dm.n_cols])
        return self._gap_ct

    def objective_and_gap(self):
        """(objective, gap) (engine.py:325-351) from the fused gap kernels."""
        self.check_solves()
        self._flush_v()
        D = _D()
        a_local = self.alpha_dev[self.col_offset:self.col_offset + self.dm.n_cols]
        ct = None
        if self.spec.coord_target is not None:
            ct = D.to_device(np.asarray(self.spec.coord_target)[
                self.col_offset:self.col_offset + self.dm.n_cols])
        L.check(L.lib().glm_gap_terms(
            ctypes.byref(self.dm.struct), self.spec.index, self.spec.lam, self.spec.l1_ratio,
            D.ptr(self.row_target), D.ptr(ct), D.ptr(a_local), D.ptr(self.v_dev),
            D.ptr(self.w_scratch), D.ptr(self.gap_out), D.ptr(D.scratch(self.stream)),
            D.sptr(self.stream)), "glm_gap_terms")
        terms = self.gap_out
        if self.reducer is not None:                 # engine.py:339-341
            stats = terms[1:3].clone()
            self.reducer.allreduce_inplace(stats)
            terms = torch.cat([terms[0:1], stats, terms[3:4]])
        h = D.to_host(terms)
        obj = float(h[3] + h[1])
        gap = float(h[0] + h[1] + h[2]) if self.spec.has_gap else None
        return obj, gap

    def train(self, stopping):
        """engine.py:353-398."""
        cfg = self.config
        trace = ConvergenceTrace()
        self.last_trace = trace
        t0 = time.perf_counter()
        per_round_cost = 0.0
        if self.cost_model is not None:
            per_round_cost = (self.cost_model.c1
                              + cfg.t2 * (self.cost_model.c2 + self.cost_model.c_comp))
        reason = "max_rounds"
        rounds = 0

        def record(rnd):
            obj, gap = self.objective_and_gap()
            trace.append(TraceRow(round=rnd, wall_s=time.perf_counter() - t0,
                                  sim_cost=rnd * per_round_cost, objective=obj, gap=gap,
                                  theta=None))
            return obj, gap

        obj, gap = record(0)
        if _met(stopping, obj, gap):
            reason = "target_met"
        else:
            max_rounds = cfg.t1 if stopping.max_rounds is None else stopping.max_rounds
            for rnd in range(1, max_rounds + 1):
                self.outer_round()
                rounds = rnd
                obj, gap = record(rnd)
                if _met(stopping, obj, gap):
                    reason = "target_met"
                    break
                if (stopping.time_budget_s is not None
                        and time.perf_counter() - t0 > stopping.time_budget_s):
                    reason = "time_budget"
                    break
        self.check_solves()
        self._flush_v()
        alpha = self.alpha_global()
        self.spec.check_alpha(alpha)
        return TrainResult(model=Model(alpha, self.spec), trace=trace, v=self.v.copy(),
                           rounds=rounds, stop_reason=reason, theta_bar_max=None,
                           theta_bars=[])

    def alpha_global(self):
        """Full alpha; in multi-process mode gathers the remote slices (engine.py:400-407)."""
        if self.reducer is None:
            return self.alpha
        padded = torch.zeros_like(self.alpha_dev)
        for wk in self.workers.values():
            padded[wk.lo:wk.hi] = self.alpha_dev[wk.lo:wk.hi]
        if self.reducer.on_cuda:
            self.reducer.allreduce_inplace(padded)
            return _D().to_host(padded).copy()
        return np.asarray(self.reducer.allreduce_sum(_D().to_host(padded)))


def _met(stopping, obj, gap):
    if stopping.target_gap is not None and gap is not None and gap <= stopping.target_gap:
        return True
    if stopping.target_subopt is not None and stopping.f_star is not None \
            and obj - stopping.f_star <= stopping.target_subopt:
        return True
    return False


def train(matrix, spec, config, stopping, **kwargs):
    """Convenience wrapper: build an Engine and run it (engine.py:420-423)."""
    return Engine(matrix, spec, config, **kwargs).train(stopping)
