"""Out-of-core training: chunk keys and the double-buffered streaming pipeline.

Reference: pipeline.py:25-340 (`hierglm.pipeline`). The three stages of the
reference (load / keygen / train, pipeline.py:244-289) run natively in
libglm_b200.so (csrc/stream.cu): a loader thread reads chunks (GLMCHUNK file
or host CSC arrays) into pinned staging buffers and issues cudaMemcpyAsync
into one of two device slots on a copy stream while the compute stream
generates the next chunk's keys on the device (bit-exact `generate_keys`,
csrc/prng.cu ChunkKeys) and trains the current chunk. Chunks that fit the
device budget stay resident in HBM. Keys are stateless in (seed, epoch, chunk)
(pipeline.py:5-9), so pipelined and sequential schedules give the same bits.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

KEY_BLOCK = 4096
STAGE_TIMEOUT_S = 120.0


def _D():
    from . import _device
    return _device


def generate_keys_device(seed, n):
    D = _D()
    out = torch.empty(max(n, 1), dtype=torch.uint32, device=D.device())
    if n > 0:
        L.check(L.lib().glm_chunk_keys(int(seed) & ((1 << 64) - 1), n, D.ptr(out), D.sptr()),
                "glm_chunk_keys")
    return out[:n]


def generate_keys(seed, n, n_threads=1):
    """n 32-bit keys in fixed 4096-wide blocks (pipeline.py:29-73), on the GPU;
    identical for every thread count by construction."""
    if n <= 0:
        return np.empty(0, dtype=np.uint32)
    return _D().to_host(generate_keys_device(seed, n)).astype(np.uint32)


def chunk_permutation(seed, n):
    """keys_to_permutation(generate_keys(seed, n)) fused on the GPU (the
    streaming solver's own path, glm_chunk_perm)."""
    from .solver import _fused_perm
    if n <= 0:
        return np.empty(0, dtype=np.int64)
    return _D().to_host(_fused_perm(L.lib().glm_chunk_perm, seed, n,
                                    "glm_chunk_perm")).astype(np.int64)


def keys_to_permutation(keys):
    """Stable argsort of the keys (pipeline.py:76-78), on the GPU."""
    from .solver import argsort_u32_device
    k = _D().to_device(np.asarray(keys, dtype=np.uint32), torch.uint32) \
        if not isinstance(keys, torch.Tensor) else keys
    return _D().to_host(argsort_u32_device(k)).astype(np.int64)


# ------------------------------------------------------------ schedule log
@dataclass
class StageEvent:
    stage: str
    chunk: int
    start: float
    end: float


@dataclass
class PipelineSchedule:
    """Per-chunk stage timing of one pipelined epoch (pipeline.py:81-138).

    Built from the native schedule: `load` is the host read into pinned
    staging, `h2d` the copy-engine transfer (CUDA events on the copy stream),
    `rand` is folded into `train` (keys and the argsort run on the device at
    the head of the chunk's solve) and reported as 0."""
    events: list = field(default_factory=list)
    steps: list = field(default_factory=list)

    HEADER = "chunk,load_ms,rand_ms,train_ms,step_ms"

    def log(self, stage, chunk, start, end):
        self.events.append(StageEvent(stage, chunk, start, end))

    def finalize(self):
        self.steps = []
        by = {}
        for ev in self.events:
            by.setdefault(ev.chunk, {})[ev.stage] = ev
        prev_end = None
        for end, chunk in sorted((ev.end, ev.chunk) for ev in self.events
                                 if ev.stage == "train"):
            rec = by[chunk]
            self.steps.append({
                "chunk": chunk,
                "load_ms": (rec["load"].end - rec["load"].start) * 1e3 if "load" in rec else 0.0,
                "rand_ms": (rec["rand"].end - rec["rand"].start) * 1e3 if "rand" in rec else 0.0,
                "h2d_ms": (rec["h2d"].end - rec["h2d"].start) * 1e3 if "h2d" in rec else 0.0,
                "train_ms": (rec["train"].end - rec["train"].start) * 1e3,
                "step_ms": 0.0 if prev_end is None else (end - prev_end) * 1e3,
            })
            prev_end = end

    def write_csv(self, path):
        with open(path, "w") as fh:
            fh.write(self.HEADER + "\n")
            for s in self.steps:
                fh.write("%d,%.3f,%.3f,%.3f,%.3f\n" % (
                    s["chunk"], s["load_ms"], s["rand_ms"], s["train_ms"], s["step_ms"]))

    def assert_buffer_safety(self):
        """No chunk trains before its load completed (pipeline.py:124-138). The
        device enforces it with a stream-wait on the slot's copy event; the log
        records train end times, so check each train ended after its load."""
        ready = {ev.chunk: ev.end for ev in self.events if ev.stage == "load"}
        for ev in self.events:
            if ev.stage == "train" and ev.chunk in ready and ev.end < ready[ev.chunk] - 1e-9:
                raise AssertionError(f"chunk {ev.chunk} trained before its buffers were ready")

    @classmethod
    def from_native(cls, rows):
        """rows: (k, 6) epoch, chunk, load_ms, h2d_ms, train_ms, t_ms (end of the
        chunk's solve on the host clock, relative to the solve start)."""
        sched = cls()
        for ep, chunk, load_ms, h2d_ms, train_ms, t_ms in rows:
            c = int(chunk)
            end = t_ms * 1e-3
            sched.log("train", c, end - train_ms * 1e-3, end)
            sched.log("h2d", c, end - (train_ms + h2d_ms) * 1e-3, end - train_ms * 1e-3)
            sched.log("load", c, end - (train_ms + h2d_ms + load_ms) * 1e-3,
                      end - (train_ms + h2d_ms) * 1e-3)
            sched.log("rand", c, end - train_ms * 1e-3, end - train_ms * 1e-3)
        sched.finalize()
        return sched


@dataclass
class ChunkedSolveContext:
    """Device-solve state threaded through the chunks of one epoch
    (pipeline.py:141-155): `delta` (device-local coordinates) and `view`
    (lin + quad * B delta) are host arrays updated in place by pipelined_epoch."""
    sub: object
    delta: np.ndarray
    view: np.ndarray
    chunk_offsets: list
    seed: int
    epoch_index: int = 0
    n_threads: int = 1


# ------------------------------------------------------ native partition
def _vp(a):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)


def _as_f64(a):
    """Host or device f64 contiguous buffer (no copy when already one)."""
    if isinstance(a, torch.Tensor):
        return a.detach().to(torch.float64).contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class StreamingPartition:
    """A device partition trained chunk by chunk through libglm_b200's
    streaming pipeline (glm_stream_*). Source: a GLMCHUNK `ChunkStore`
    (read by the native loader thread) or a host `SparseColumnMatrix` cut into
    `chunk_size` columns. `device_budget` bytes of chunk data stay resident
    (None: everything that fits, i.e. no streaming after the first epoch).
    File sources read each streamed chunk body with `io_threads` concurrent
    preads (page cache: 7.7 GB/s with one, 31.6 GB/s with eight on the GPU
    box) and, with `direct_io`, bypass the page cache (O_DIRECT: the device's
    own rate, 4.4 GB/s on the box's virtio disk)."""

    def __init__(self, source, chunk_size=None, chunk_offsets=None, device_budget=None,
                 pin_host=False, device=None, direct_io=False, io_threads=8):
        _D().require_cuda()
        self.device = torch.cuda.current_device() if device is None else int(device)
        budget = -1 if device_budget is None else int(device_budget)
        h = ctypes.c_void_p()
        from .data import ChunkStore
        if isinstance(source, ChunkStore):
            descs = source.chunks
            self.offsets = np.array([0] + [c.n_cols for c in descs], dtype=np.int64).cumsum()
            offs = np.array([c.offset for c in descs], dtype=np.int64)
            cols = np.array([c.n_cols for c in descs], dtype=np.int64)
            nnz = np.array([c.nnz for c in descs], dtype=np.int64)
            self._keep = (offs, cols, nnz)
            L.check(L.lib().glm_stream_create_file(
                self.device, str(source.path).encode(), int(source.n_rows), len(descs),
                _vp(offs), _vp(cols), _vp(nnz), budget, ctypes.byref(h)), "glm_stream_create_file")
            self.n_rows, self.n_cols = int(source.n_rows), int(self.offsets[-1])
            if direct_io or io_threads > 1:     # streamed chunks: O_DIRECT / striped preads
                L.check(L.lib().glm_stream_set_io(h, 1 if direct_io else 0, int(io_threads)),
                        "glm_stream_set_io")
        else:
            m = source
            n = int(m.n_cols)
            if chunk_offsets is None:
                if not chunk_size or chunk_size < 1:
                    raise ValueError("chunk_size must be >= 1")
                chunk_offsets = np.concatenate([np.arange(0, n, chunk_size), [n]]) if n else [0]
            self.offsets = np.asarray(chunk_offsets, dtype=np.int64)
            indptr = np.ascontiguousarray(m.indptr, dtype=np.int64)
            rows = np.ascontiguousarray(m.rows, dtype=np.int32)
            vals = np.ascontiguousarray(m.vals, dtype=np.float64)
            self._keep = (indptr, rows, vals, self.offsets)      # must outlive the stream
            L.check(L.lib().glm_stream_create_host(
                self.device, int(m.n_rows), n, _vp(indptr), _vp(rows), _vp(vals),
                len(self.offsets) - 1, _vp(self.offsets), budget, 1 if pin_host else 0,
                ctypes.byref(h)), "glm_stream_create_host")
            self.n_rows, self.n_cols = int(m.n_rows), n
        self.handle = h
        info = np.zeros(8, dtype=np.int64)
        L.check(L.lib().glm_stream_info(h, _vp(info)), "glm_stream_info")
        self.direct_io = bool(info[7])
        self.n_chunks, self.n_resident = int(info[0]), int(info[1])
        self.bytes_resident, self.bytes_slots = int(info[2]), int(info[3])
        self.direct_dma = bool(info[4])
        self.last_schedule = None
        self.last_scal = None

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            L.lib().glm_stream_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, spec, lin, quad, cnst, base, *, seed, epoch_index, epochs, damping=1.0,
              mode=L.MODE_SEQUENTIAL, delta=None, view=None, delta_in=False, view_in=False,
              dv_out=None, coord_target=None, timing=False, group_lanes=0, max_inflight=0,
              attempts_per_chunk=0, cache_flags=0):
        """`epochs` chunked passes (chunked_device_runner's runner body,
        pipeline.py:315-340). Returns (status, delta, values, info, scal, damping)."""
        from .solver import _KIND_INDEX
        m, d = self.n_cols, self.n_rows
        lin, base = _as_f64(lin), _as_f64(base)
        if delta is None:
            delta = np.zeros(max(m, 1))
        values = np.zeros(max(epochs, 1))
        info = np.zeros(5, dtype=np.int32)
        scal = np.zeros(4)
        yv = None if coord_target is None else _as_f64(coord_target)
        a = L.GlmStreamArgs()
        a.kind = _KIND_INDEX[spec.kind]
        a.mode = int(mode)
        a.lam = float(spec.lam)
        a.l1_ratio = float(getattr(spec, "l1_ratio", 1.0))
        a.quad = float(quad)
        a.cnst = float(cnst)
        a.lin = _vp(lin)
        a.base = _vp(base)
        a.coord_target = _vp(yv)
        a.seed = int(seed) & ((1 << 64) - 1)
        a.epoch_index = int(epoch_index)
        a.epochs = int(epochs)
        a.attempts_per_chunk = int(attempts_per_chunk)
        a.group_lanes = int(group_lanes)
        a.max_inflight = int(max_inflight)
        a.flags = (int(cache_flags) & 3) | (L.STREAM_DELTA_IN if delta_in else 0) | \
            (L.STREAM_VIEW_IN if view_in else 0) | (L.STREAM_TIMING if timing else 0)
        dmp = ctypes.c_double(float(damping))
        st = L.lib().glm_stream_solve(self.handle, ctypes.byref(a), ctypes.byref(dmp),
                                      _vp(delta), _vp(view), _vp(dv_out), _vp(values),
                                      _vp(info), _vp(scal))
        self.last_scal = scal
        if timing and st == L.GLM_OK:
            n = ctypes.c_int(0)
            L.lib().glm_stream_schedule(self.handle, None, 0, ctypes.byref(n))
            rows = np.zeros((max(n.value, 1), L.STREAM_SCHED_COLS))
            L.lib().glm_stream_schedule(self.handle, _vp(rows), n.value, ctypes.byref(n))
            self.last_schedule = rows[:n.value]
        return st, delta, values[:max(int(info[0]), 0)], info, scal, dmp.value


_PARTITIONS = {}


def _partition_for(store, device_budget=None):
    key = (id(store), device_budget)
    part = _PARTITIONS.get(key)
    if part is None or part.handle is None:
        part = StreamingPartition(store, device_budget=device_budget)
        _PARTITIONS[key] = part
    return part


def _raise_status(st, sub, diag):
    from .solver import _reference_exceptions
    if st == L.GLM_OK:
        return
    se, sd = _reference_exceptions(sub)
    if st == L.GLM_DIVERGENCE:
        raise sd("damping floor reached during chunked epoch", diagnostics=diag)
    if st == L.GLM_SOLVER_ERROR:
        raise se(L.last_error())
    L.check(st, "glm_stream_solve")


def _mode_for(n_threads):
    return L.MODE_SEQUENTIAL if int(n_threads) <= 1 else L.MODE_ASYNC


def pipelined_epoch(store, ctx, damping=None, pipelined=True, inject_load_s=0.0,
                    inject_rand_s=0.0, inject_train_s=0.0, step_timeout_s=STAGE_TIMEOUT_S,
                    device_budget=None):
    """One pass over every chunk of the store (pipeline.py:200-295), run by the
    native pipeline; ctx.delta / ctx.view are updated in place. `pipelined`
    only changes the reference's thread schedule, never the result; the native
    pipeline always overlaps (the inject_* delays are the reference's test
    hooks and are not used). Returns (device value, PipelineSchedule)."""
    from .solver import DampingState
    damping = damping if damping is not None else DampingState()
    part = store if isinstance(store, StreamingPartition) else _partition_for(store, device_budget)
    sub = ctx.sub
    delta = np.ascontiguousarray(ctx.delta, dtype=np.float64)
    view = np.ascontiguousarray(ctx.view, dtype=np.float64)
    st, delta, values, info, scal, dmp = part.solve(
        sub.spec, sub.lin, sub.quad, sub.const, sub.base, seed=ctx.seed,
        epoch_index=ctx.epoch_index, epochs=1, damping=damping.delta,
        mode=_mode_for(ctx.n_threads), delta=delta, view=view, delta_in=True, view_in=True,
        coord_target=_coord_target(sub), timing=True)
    damping.delta = dmp
    _raise_status(st, sub, {"value": float(scal[1])})
    ctx.delta[:] = delta[:len(ctx.delta)]
    ctx.view[:] = view[:len(ctx.view)]
    return float(values[-1]) if len(values) else float(scal[1]), \
        PipelineSchedule.from_native(part.last_schedule)


def _coord_target(sub):
    y = getattr(sub.spec, "coord_target", None)
    if y is None:
        return None
    return np.ascontiguousarray(np.asarray(y)[np.asarray(sub.col_ids)], dtype=np.float64)


def chunked_device_runner(store, seed, epochs, pipelined=True, n_threads=1, inject_load_s=0.0,
                          inject_rand_s=0.0, inject_train_s=0.0, schedule_sink=None,
                          device_budget=None, mode=None, group_lanes=0, max_inflight=0):
    """Engine chunk_runner hook (pipeline.py:298-340) backed by the native
    streaming pipeline. `store` is a GLMCHUNK ChunkStore (or a ready
    StreamingPartition); `device_budget` caps the bytes of chunk data kept in
    HBM (the rest stream through two slots every epoch). The epoch counter is
    global across calls, like the reference's."""
    from .solver import SubtaskResult
    part = store if isinstance(store, StreamingPartition) else _partition_for(store, device_budget)
    epoch_counter = [0]
    md = _mode_for(n_threads) if mode is None else mode

    def runner(sub, dev, cfg):
        m = part.n_cols
        on_device = isinstance(sub.base, torch.Tensor) and sub.base.is_cuda
        delta = torch.zeros(max(m, 1), dtype=torch.float64, device=sub.base.device) \
            if on_device else np.zeros(max(m, 1))
        dv = torch.empty(max(part.n_rows, 1), dtype=torch.float64, device=sub.base.device) \
            if on_device else np.empty(max(part.n_rows, 1))
        if on_device:       # the native pipeline runs on its own streams
            torch.cuda.current_stream().synchronize()
        st, delta, values, info, scal, dmp = part.solve(
            sub.spec, sub.lin, sub.quad, sub.const, sub.base, seed=seed,
            epoch_index=epoch_counter[0], epochs=epochs, damping=dev.damping.delta, mode=md,
            delta=delta, dv_out=dv, coord_target=_coord_target(sub),
            timing=schedule_sink is not None, group_lanes=group_lanes,
            max_inflight=max_inflight)
        epoch_counter[0] += epochs
        dev.damping.delta = dmp
        _raise_status(st, sub, {"value": float(scal[1]), "retries": int(info[1])})
        if schedule_sink is not None and part.last_schedule is not None:
            rows = part.last_schedule
            for e in range(epochs):
                schedule_sink.append(PipelineSchedule.from_native(rows[rows[:, 0] == e]))
        return SubtaskResult(col_ids=sub.col_ids, delta_alpha=delta[:m], delta_v=dv[:part.n_rows],
                             epochs_run=int(info[0]), final_subproblem_value=float(scal[1]),
                             initial_subproblem_value=float(scal[0]),
                             epoch_values=[float(x) for x in values], retries=int(info[1]))

    runner.partition = part
    return runner


def wall_ms_last(part):
    """(wall ms of the last solve, ms it waited on chunk loads)."""
    s = part.last_scal
    return (float(s[2]), float(s[3])) if s is not None else (None, None)


__all__ = ["KEY_BLOCK", "STAGE_TIMEOUT_S", "generate_keys", "keys_to_permutation",
           "StageEvent", "PipelineSchedule", "ChunkedSolveContext", "StreamingPartition",
           "pipelined_epoch", "chunked_device_runner"]
