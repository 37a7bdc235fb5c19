"""Device plumbing: torch owns HBM allocations and streams; every kernel is
launched through the C-ABI (libglm_b200.so). No CPU fallback exists — any call
without a CUDA device raises."""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib as L

F64 = torch.float64
_scratch = {}
_scratch_lock = threading.Lock()


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1803_06333_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    L.load()


def device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def sptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def to_device(x, dtype=F64):
    """numpy / list / torch -> contiguous CUDA tensor of `dtype` (copy if needed)."""
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == dtype and x.is_contiguous():
            return x
        return x.to(device=device(), dtype=dtype).contiguous()
    np_dtype = {torch.float64: np.float64, torch.int64: np.int64, torch.int32: np.int32,
                torch.uint32: np.uint32, torch.uint64: np.uint64}[dtype]
    arr = np.ascontiguousarray(np.asarray(x, dtype=np_dtype))
    return torch.from_numpy(arr).to(device())


def to_host(t):
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def scratch(stream=None):
    """Zeroed reduction scratch private to (device, stream)."""
    s = stream if stream is not None else torch.cuda.current_stream()
    key = (torch.cuda.current_device(), s.cuda_stream)
    with _scratch_lock:
        buf = _scratch.get(key)
        if buf is None:
            nbytes = L.lib().glm_reduce_scratch_bytes()
            buf = torch.zeros(nbytes // 8 + 8, dtype=F64, device=device())
            _scratch[key] = buf
        return buf


def fgrad(spec, v, tgt=None, want_grad=True, stream=None):
    """(f'(v) tensor or None, f(v) float) — fused kernel, reads back one scalar."""
    out = torch.empty(1, dtype=F64, device=v.device)
    grad = torch.empty_like(v) if want_grad else None
    L.check(L.lib().glm_fgrad(spec.index, spec.lam, ptr(tgt), ptr(v), v.numel(), ptr(grad),
                              ptr(out), ptr(scratch(stream)), sptr(stream)), "glm_fgrad")
    return grad, float(out.item())


def gsum(spec, a, y=None, stream=None):
    out = torch.empty(1, dtype=F64, device=a.device)
    L.check(L.lib().glm_gsum(spec.index, spec.lam, spec.l1_ratio, ptr(y), ptr(a), a.numel(),
                             ptr(out), ptr(scratch(stream)), sptr(stream)), "glm_gsum")
    return float(out.item())


def gap_terms(spec, dm, alpha, v, stream=None, out=None):
    """[f(v)+f*(w), sum g(alpha), sum g*(-A^T w), f(v)] over DeviceMatrix dm."""
    a = to_device(alpha)
    vv = to_device(v)
    tgt = to_device(spec.row_target) if spec.row_target is not None else None
    y = to_device(spec.coord_target) if spec.coord_target is not None else None
    w = torch.empty_like(vv)
    res = out if out is not None else torch.empty(4, dtype=F64, device=vv.device)
    L.check(L.lib().glm_gap_terms(ctypes.byref(dm.struct), spec.index, spec.lam, spec.l1_ratio,
                                  ptr(tgt), ptr(y), ptr(a), ptr(vv), ptr(w), ptr(res),
                                  ptr(scratch(stream)), sptr(stream)), "glm_gap_terms")
    if out is not None:
        return out
    return to_host(res)
