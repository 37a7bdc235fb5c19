"""Shared-vector reducers: the reference's Reducer duck type over NCCL.

Reference: comm.py:41-114 (canonical_sum, InProcessReducer, participant API:
allreduce_sum / broadcast / handshake / abort / close) and comm.py:437-444
(make_reducer). The TCP star/ring reducers (comm.py:117-434) are replaced by
NCCL over NVLink 5 / NVSwitch through torch.distributed: one process per GPU.

* `NcclReducer(deterministic=False)`: allreduce_sum is one ncclAllReduce
  (f64, sum) — identical on every rank, summation order chosen by NCCL.
* `NcclReducer(deterministic=True)`: ncclAllGather + a fold in ascending rank
  order, bit-identical to canonical_sum (comm.py:41-46).
Both accept CUDA tensors (device-resident engine) or numpy arrays.
`make_reducer("gloo", ...)` gives the same semantics on CPU tensors for the
multi-process tests without a GPU.
"""

from __future__ import annotations

import threading

import numpy as np
import torch
import torch.distributed as dist

PROTOCOL_VERSION = 1


class ReduceError(RuntimeError):
    pass


class ProtocolError(ReduceError):
    pass


def canonical_sum(vectors):
    """Left-fold sum in ascending rank order (comm.py:41-46)."""
    out = vectors[0].clone() if isinstance(vectors[0], torch.Tensor) else vectors[0].copy()
    for vec in vectors[1:]:
        out += vec
    return out


class InProcessReducer:
    """Collective sum across `world` threads of one process (comm.py:53-63)."""

    def __init__(self, world):
        self.world = world
        self._barrier = threading.Barrier(world)
        self._slots = [None] * world
        self._result = None

    def participant(self, rank):
        return _InProcessParticipant(self, rank)


class _InProcessParticipant:
    topology = "in_process"

    def __init__(self, owner, rank):
        self.owner = owner
        self.rank = rank

    def handshake(self):
        return {"rank": self.rank, "world": self.owner.world, "version": PROTOCOL_VERSION}

    def _wait(self):
        try:
            self.owner._barrier.wait()
        except threading.BrokenBarrierError:
            raise ReduceError("collective aborted by a peer") from None

    def allreduce_sum(self, vec):
        owner = self.owner
        owner._slots[self.rank] = vec
        self._wait()
        if self.rank == 0:
            lengths = {len(s) for s in owner._slots}
            owner._result = ProtocolError("vector length mismatch") if len(lengths) != 1 \
                else canonical_sum(owner._slots)
        self._wait()
        result = owner._result
        self._wait()
        if isinstance(result, Exception):
            raise result
        return result.clone() if isinstance(result, torch.Tensor) else result.copy()

    def broadcast(self, vec):
        owner = self.owner
        if self.rank == 0:
            owner._result = vec
        self._wait()
        result = owner._result
        self._wait()
        return result.clone() if isinstance(result, torch.Tensor) else np.array(result)

    def abort(self):
        self.owner._barrier.abort()

    def close(self):
        pass


class NcclReducer:
    """Reducer duck type over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    topology = "nccl"

    def __init__(self, group=None, deterministic=False, device=None):
        if not dist.is_initialized():
            raise ReduceError("torch.distributed is not initialised")
        self.group = group
        self.deterministic = deterministic
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.on_cuda = backend == "nccl"
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if self.on_cuda
            else torch.device("cpu"))
        # gloo: device tensors are staged through host memory (several ranks
        # may then share one GPU, which NCCL refuses)
        self.staged = not self.on_cuda
        self._aborted = False
        self._hbuf = None          # reusable device buffer for host vectors (NCCL)
        self._chk = None           # the length check's [n, -n], device + pinned host

    def handshake(self):
        probe = torch.tensor([self.rank, PROTOCOL_VERSION], dtype=torch.float64,
                             device=self.device)
        got = [torch.empty_like(probe) for _ in range(self.world)]
        dist.all_gather(got, probe, group=self.group)
        ranks = sorted(int(g[0].item()) for g in got)
        if ranks != list(range(self.world)) or any(int(g[1].item()) != PROTOCOL_VERSION
                                                   for g in got):
            raise ProtocolError("handshake mismatch")
        return {"rank": self.rank, "world": self.world, "version": PROTOCOL_VERSION}

    def _tensor(self, vec):
        if isinstance(vec, torch.Tensor):
            return vec.to(self.device, torch.float64).contiguous(), True
        return torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64)).to(self.device), False

    def _allreduce_host(self, vec, out):
        """A host vector through NCCL: one reusable device buffer, copies from
        and to page-locked arrays asynchronous, the length check's collective
        queued behind the upload (one host synchronisation before the data
        collective, one after the download)."""
        src = np.ascontiguousarray(vec, dtype=np.float64)
        n = int(src.size)
        if self._hbuf is None or self._hbuf.numel() != n:
            self._hbuf = torch.empty(n, dtype=torch.float64, device=self.device)
        buf = self._hbuf
        h = torch.from_numpy(src)
        buf.copy_(h, non_blocking=h.is_pinned())
        if self.world > 1:          # max(n) == -max(-n), as allreduce_sum checks it
            if self._chk is None:
                self._chk = (torch.empty(2, dtype=torch.int64, device=self.device),
                             torch.empty(2, dtype=torch.int64, pin_memory=True))
            dchk, hchk = self._chk
            hchk[0], hchk[1] = n, -n
            dchk.copy_(hchk, non_blocking=True)
            dist.all_reduce(dchk, op=dist.ReduceOp.MAX, group=self.group)
            hi, neg_lo = dchk.tolist()
            if hi != -neg_lo:
                raise ProtocolError("vector length mismatch")
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
        dst = out if out is not None else np.empty(n, dtype=np.float64)
        hd = torch.from_numpy(dst)
        pinned = hd.is_pinned()
        hd.copy_(buf, non_blocking=pinned)
        if pinned:
            torch.cuda.current_stream(self.device).synchronize()
        return dst

    def allreduce_sum(self, vec, out=None):
        if self._aborted:
            raise ReduceError("collective aborted")
        if (isinstance(vec, np.ndarray) and not self.deterministic and not self.staged
                and (out is None or (isinstance(out, np.ndarray) and out.dtype == np.float64
                                     and out.flags.c_contiguous))):
            return self._allreduce_host(vec, out)
        t, was_tensor = self._tensor(vec)
        if self.world > 1:     # one collective checks the lengths: max(n) == -max(-n)
            n = torch.tensor([t.numel(), -t.numel()], dtype=torch.int64, device=self.device)
            dist.all_reduce(n, op=dist.ReduceOp.MAX, group=self.group)
            hi, neg_lo = n.tolist()
            if hi != -neg_lo:
                raise ProtocolError("vector length mismatch")
        if self.deterministic and self.staged:
            h = t.cpu()
            got = [torch.empty_like(h) for _ in range(self.world)]
            dist.all_gather(got, h, group=self.group)
            res = canonical_sum(got).to(t.device)                  # ascending rank order
        elif self.deterministic:
            flat = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(flat, t, group=self.group)
            res = canonical_sum(list(flat.view(self.world, -1)))   # ascending rank order
        elif self.staged and t.is_cuda:
            res = t.cpu()
            dist.all_reduce(res, op=dist.ReduceOp.SUM, group=self.group)
            res = res.to(t.device)
        else:
            res = t.clone()
            dist.all_reduce(res, op=dist.ReduceOp.SUM, group=self.group)
        if out is not None:
            if isinstance(out, np.ndarray):
                torch.from_numpy(out).copy_(res)
            else:
                out.copy_(res)
            return out
        return res.to(vec.device) if was_tensor else res.cpu().numpy()

    def allreduce_inplace(self, t):
        """Fast path for device-resident engines: sum into `t` (NCCL)."""
        if self._aborted:
            raise ReduceError("collective aborted")
        if self.deterministic:
            t.copy_(self.allreduce_sum(t))
        elif self.staged and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def allgather(self, t):
        """Every rank's tensor, in rank order (the parts of canonical_sum)."""
        if self._aborted:
            raise ReduceError("collective aborted")
        if self.staged:
            h = t.cpu()
            got = [torch.empty_like(h) for _ in range(self.world)]
            dist.all_gather(got, h, group=self.group)
            return [g.to(t.device) for g in got]
        flat = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(flat, t.contiguous(), group=self.group)
        return list(flat.view(self.world, -1))

    def broadcast(self, vec):
        t, was_tensor = self._tensor(vec)
        t = t.clone()
        dist.broadcast(t, src=0 if self.group is None else dist.get_global_rank(self.group, 0),
                       group=self.group)
        return t if was_tensor else t.cpu().numpy()

    def barrier(self):
        dist.barrier(group=self.group)

    def abort(self):
        self._aborted = True

    def close(self):
        pass


def make_reducer(kind="nccl", rank=None, peers=None, dim=None, deterministic=False):
    """Factory (comm.py:437-444): 'nccl' | 'gloo' use the initialised process
    group; 'inproc' returns a single-participant in-process reducer."""
    if kind in ("nccl", "gloo"):
        return NcclReducer(deterministic=deterministic)
    if kind == "inproc":
        return InProcessReducer(1).participant(0)
    raise ValueError(f"unknown reducer {kind!r} (TCP reducers are replaced by NCCL)")


class PeerExchange:
    """The round's Delta v exchange over NVLink peer memory (csrc/peer.cu):
    every rank's Delta v stays in its own HBM, mapped into every peer with
    CUDA IPC; `glm_round_start` sums the ranks' buffers in ascending rank order
    (the bits of canonical_sum on every rank, comm.py:41-46) fused with
    v += total and the next round's model. World 1 works without IPC.

    Construction is collective and agreed: every rank joins both exchanges
    (handles, then the open results) even after a local failure, and if any
    rank failed every rank closes and raises ReduceError — so all ranks fall
    back to the NCCL path together.  Every device-side wait has a deadline
    (`timeout`, default the reference's DEFAULT_TIMEOUT = 60 s, comm.py:30);
    `check()` raises ReduceError when one expired (a dead or stalled peer)."""

    DEFAULT_TIMEOUT = 60.0

    def __init__(self, d, group=None, local=False, timeout=None):
        import ctypes

        from . import _lib as L
        self.L = L
        self.handle = None
        multi = dist.is_initialized() and not local
        self.world = dist.get_world_size(group) if multi else 1
        self.rank = dist.get_rank(group) if multi else 0
        self.d = int(d)
        self.timeout = float(self.DEFAULT_TIMEOUT if timeout is None else timeout)
        h = ctypes.c_void_p()
        err = None
        mine = b""
        try:
            L.check(L.lib().glm_peer_create(torch.cuda.current_device(), self.d, self.rank,
                                            self.world, ctypes.byref(h)), "glm_peer_create")
            self.handle = h
            L.check(L.lib().glm_peer_set_timeout(h, self.timeout), "glm_peer_set_timeout")
            if self.world > 1:
                nb = int(L.lib().glm_peer_handle_bytes())
                buf = (ctypes.c_char * nb)()
                L.check(L.lib().glm_peer_handle(h, buf), "glm_peer_handle")
                mine = bytes(buf)
        except Exception as exc:          # still join the collectives below
            err = exc
        if self.world > 1:
            got = [None] * self.world
            dist.all_gather_object(got, (err is None, mine), group=group)
            if err is None and not all(ok for ok, _ in got):
                err = ReduceError("peer exchange: another rank could not create its buffers")
            if err is None:
                try:
                    L.check(L.lib().glm_peer_open(h, ctypes.c_char_p(b"".join(b for _, b in got))),
                            "glm_peer_open")
                except Exception as exc:
                    err = exc
            oks = [None] * self.world
            dist.all_gather_object(oks, err is None, group=group)
            if err is None and not all(oks):
                err = ReduceError("peer exchange: another rank could not map the buffers")
        if err is not None:
            self.close()
            if isinstance(err, ReduceError):
                raise err
            raise ReduceError(f"peer exchange unavailable: {err}") from err

    def check(self):
        """Raise ReduceError if a device-side wait ran past the deadline
        (synchronises the device)."""
        import ctypes
        code = ctypes.c_int64(0)
        self.L.check(self.L.lib().glm_peer_error(self.handle, ctypes.byref(code), 0),
                     "glm_peer_error")
        c = code.value
        if c:
            kind, what = c >> 32, c & 0xFFFFFFFF
            if kind == 1:
                raise ReduceError(f"peer exchange: rank {what} did not publish its Delta v "
                                  f"within {self.timeout:g} s (dead or stalled peer)")
            raise ReduceError(f"peer exchange: round_turn blocks were not co-resident "
                              f"(wait {what} expired after {self.timeout:g} s)")

    def consume(self, stream):
        from . import _device as D
        self.L.check(self.L.lib().glm_peer_consume(self.handle, D.sptr(stream)),
                     "glm_peer_consume")

    def close(self):
        if getattr(self, "handle", None) is not None:
            self.L.lib().glm_peer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shutdown(*engines):
    """Orderly end of a (multi-process) run: close the engines' peer exchanges,
    synchronise, and tear the process group down on every rank together, so
    the interpreter exits normally (atexit hooks run)."""
    for eng in engines:
        if eng is not None and hasattr(eng, "close"):
            eng.close()
    if torch.cuda.is_available() and torch.cuda.is_initialized():
        torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
