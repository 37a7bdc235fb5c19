"""ctypes binding of libglm_b200.so (include/glm_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, `lib()` raises. Status codes map onto the reference's
exception types (solver.py:31-38).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libglm_b200.so")

GLM_OK, GLM_SOLVER_ERROR, GLM_DIVERGENCE, GLM_USAGE, GLM_CUDA_ERROR = range(5)
CSC, DENSE = 0, 1
MODE_SEQUENTIAL, MODE_ASYNC = 0, 1
FLAG_REUSE_GSUM = 4
FLAG_PREFETCH_PERM = 8
FLAG_PEER_FINALIZE = 32
FLAG_SKIP_BEGIN = 64
FLAG_TURN = 128
STREAM_DELTA_IN, STREAM_VIEW_IN, STREAM_TIMING = 16, 32, 64
STREAM_SCHED_COLS = 6

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_c_dbl = ctypes.c_double
_c_u64 = ctypes.c_uint64
_P = ctypes.c_void_p


class GlmMatrix(ctypes.Structure):
    _fields_ = [("n_rows", _c_i64), ("n_cols", _c_i64), ("nnz", _c_i64), ("layout", _c_i32),
                ("_pad", _c_i32), ("indptr", _P), ("rows", _P), ("vals", _P), ("sqnorms", _P)]


class GlmSolveArgs(ctypes.Structure):
    _fields_ = [("kind", _c_i32), ("mode", _c_i32), ("lam", _c_dbl), ("l1_ratio", _c_dbl),
                ("quad", _c_dbl), ("cnst", _P), ("lin", _P), ("base", _P),
                ("coord_target", _P), ("epochs", _c_i32), ("max_attempts", _c_i32),
                ("group_lanes", _c_i32), ("max_inflight", _c_i32), ("reset_damping", _c_i32),
                ("accumulate", _c_i32), ("flags", _c_i32), ("peer", _P)]


class GlmSolveResult(ctypes.Structure):
    _fields_ = [("status", _c_i32), ("epochs_run", _c_i32), ("retries", _c_i32),
                ("plateaued", _c_i32), ("attempts", _c_i32), ("done", _c_i32),
                ("damping", _c_dbl), ("initial_value", _c_dbl), ("final_value", _c_dbl),
                ("gen_state", _c_u64)]


class GlmStreamArgs(ctypes.Structure):
    _fields_ = [("kind", _c_i32), ("mode", _c_i32), ("lam", _c_dbl), ("l1_ratio", _c_dbl),
                ("quad", _c_dbl), ("cnst", _c_dbl), ("lin", _P), ("base", _P),
                ("coord_target", _P), ("seed", _c_u64), ("epoch_index", _c_u64),
                ("epochs", _c_i32), ("attempts_per_chunk", _c_i32), ("group_lanes", _c_i32),
                ("max_inflight", _c_i32), ("flags", _c_i32), ("_pad", _c_i32)]


# name -> (restype, argtypes); every symbol of include/glm_b200.h
SIGNATURES = {
    "glm_last_error": (ctypes.c_char_p, []),
    "glm_version": (ctypes.c_int, []),
    "glm_launch_count": (ctypes.c_longlong, []),
    "glm_solver_timing": (ctypes.c_int, [_P, ctypes.c_int]),
    "glm_solver_timing_read": (ctypes.c_int, [_P, _P, _P]),
    "glm_solver_timing_peek": (ctypes.c_int, [_P, _P, _P]),
    "glm_solver_timing_glue": (ctypes.c_int, [_P, _P, _P, ctypes.c_int]),
    "glm_device_count": (ctypes.c_int, [_P]),
    "glm_debug_timeline": (ctypes.c_int, [_P]),
    "glm_xorshift_jump": (_c_u64, [_c_u64, _c_u64]),
    "glm_derive_seed": (_c_u64, [_c_u64, _P, ctypes.c_int]),
    "glm_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _c_i64, _c_i64, _P, _P, _P, _P]),
    "glm_ctx_destroy": (ctypes.c_int, [_P]),
    "glm_device_solve": (ctypes.c_int, [_P, ctypes.c_int, _c_dbl, _c_dbl, _P, _P, _c_dbl, _c_dbl,
                                        _P, _P, _P, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P,
                                        _P]),
    "glm_ctx_gap_terms": (ctypes.c_int, [_P, ctypes.c_int, _c_dbl, _c_dbl, _P, _P, _P, _P, _P]),
    "glm_solver_create": (ctypes.c_int, [ctypes.c_int, _c_i64, _c_i64, _P]),
    "glm_solver_destroy": (ctypes.c_int, [_P]),
    "glm_solver_set_state": (ctypes.c_int, [_P, _c_u64, _c_dbl, _P]),
    "glm_solve": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "glm_solver_result": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, _P]),
    "glm_solver_join": (ctypes.c_int, [_P, _P]),
    "glm_perm_keys": (ctypes.c_int, [_c_u64, _c_i64, _P, _P]),
    "glm_chunk_keys": (ctypes.c_int, [_c_u64, _c_i64, _P, _P]),
    "glm_argsort_temp_bytes": (ctypes.c_size_t, [_c_i64]),
    "glm_argsort_u32": (ctypes.c_int, [_P, _c_i64, _P, _P, ctypes.c_size_t, _P]),
    "glm_perm": (ctypes.c_int, [_c_u64, _c_i64, _P, _P, ctypes.c_size_t, _P]),
    "glm_chunk_perm": (ctypes.c_int, [_c_u64, _c_i64, _P, _P, ctypes.c_size_t, _P]),
    "glm_col_sqnorms": (ctypes.c_int, [_P, _P, _P]),
    "glm_matvec": (ctypes.c_int, [_P, _P, _P, _P]),
    "glm_rmatvec": (ctypes.c_int, [_P, _P, _P, _P]),
    "glm_transpose_temp_bytes": (ctypes.c_size_t, [_c_i64, _c_i64]),
    "glm_transpose": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "glm_select_temp_bytes": (ctypes.c_size_t, [_c_i64]),
    "glm_select_indptr": (ctypes.c_int, [_P, _P, _c_i64, _P, _P, ctypes.c_size_t, _P]),
    "glm_select_gather": (ctypes.c_int, [_P, _P, _c_i64, _P, _P, _P, _P]),
    "glm_scale_columns": (ctypes.c_int, [_P, _P, _P, _P]),
    "glm_validate": (ctypes.c_int, [_P, _P]),
    "glm_reduce_scratch_bytes": (ctypes.c_size_t, []),
    "glm_fgrad": (ctypes.c_int, [ctypes.c_int, _c_dbl, _P, _P, _c_i64, _P, _P, _P, _P]),
    "glm_outer_model": (ctypes.c_int, [ctypes.c_int, _c_dbl, _P, _P, _c_i64, _P, _P, _P, _P,
                                       _c_dbl, _c_dbl, _P, _P]),
    "glm_inner_model": (ctypes.c_int, [_P, _P, _c_i64, _c_dbl, _P, _c_dbl, _c_dbl, _P, _P, _P,
                                       _P]),
    "glm_axpby": (ctypes.c_int, [_c_i64, _c_dbl, _P, _c_dbl, _P, _P]),
    "glm_gap_terms": (ctypes.c_int, [_P, ctypes.c_int, _c_dbl, _c_dbl, _P, _P, _P, _P, _P, _P,
                                     _P, _P]),
    "glm_gsum": (ctypes.c_int, [ctypes.c_int, _c_dbl, _c_dbl, _P, _P, _c_i64, _P, _P, _P]),
    "glm_predict": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, _P, _P, _P, _P, _P]),
    "glm_coordinate_steps": (ctypes.c_int, [ctypes.c_int, _c_dbl, _c_dbl, _P, _P, _P, _P, _c_i64,
                                            _P, _P]),
    "glm_stream_create_host": (ctypes.c_int, [ctypes.c_int, _c_i64, _c_i64, _P, _P, _P,
                                              ctypes.c_int, _P, _c_i64, ctypes.c_int, _P]),
    "glm_stream_create_file": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, _c_i64, ctypes.c_int,
                                              _P, _P, _P, _c_i64, _P]),
    "glm_stream_destroy": (ctypes.c_int, [_P]),
    "glm_stream_info": (ctypes.c_int, [_P, _P]),
    "glm_stream_set_io": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int]),
    "glm_stream_solve": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "glm_stream_schedule": (ctypes.c_int, [_P, _P, ctypes.c_int, _P]),
    "glm_peer_create": (ctypes.c_int, [ctypes.c_int, _c_i64, ctypes.c_int, ctypes.c_int, _P]),
    "glm_peer_handle_bytes": (ctypes.c_size_t, []),
    "glm_peer_handle": (ctypes.c_int, [_P, _P]),
    "glm_peer_open": (ctypes.c_int, [_P, _P]),
    "glm_peer_consume": (ctypes.c_int, [_P, _P]),
    "glm_round_start": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, _c_dbl, _P, _P, _c_i64,
                                       _P, _P, _P, _P, _c_dbl, _c_dbl, ctypes.c_int, _P, _P]),
    "glm_peer_destroy": (ctypes.c_int, [_P]),
    "glm_peer_stamps": (ctypes.c_int, [_P, _P]),
    "glm_peer_set_timeout": (ctypes.c_int, [_P, ctypes.c_double]),
    "glm_solver_prepare": (ctypes.c_int, [_P, _P, _P]),
    "glm_peer_error": (ctypes.c_int, [_P, _P, ctypes.c_int]),
    "glm_round_turn": (ctypes.c_int, [_P, _P, ctypes.c_int, _c_dbl, _c_dbl, _P, _P, _c_i64, _P,
                                      _P, _c_i64, _P, _P, _P, _c_dbl, _c_dbl, ctypes.c_int, _P,
                                      _P]),
    "glm_svmlight_parse": (ctypes.c_int, [_P, _c_i64, ctypes.c_int, _P, _P]),
    "glm_svmlight_fetch": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "glm_svmlight_free": (ctypes.c_int, [_P]),
    "glm_chunk_write": (ctypes.c_int, [ctypes.c_char_p, _c_i64, _c_i64, _P, _P, _P, _P, _P,
                                       _c_i64, _P, _P]),
    "glm_chunk_open": (ctypes.c_int, [ctypes.c_char_p, _P, _P, _P]),
    "glm_chunk_table": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "glm_chunk_close": (ctypes.c_int, [_P]),
    "glm_chunk_read": (ctypes.c_int, [ctypes.c_char_p, _c_i64, _c_i64, _c_i64, ctypes.c_int,
                                      _P, _P, _P, _P, _P]),
}

_LIB = None
_LOCK = threading.Lock()


class GlmCudaError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load the shared library and bind every exported symbol (no GPU needed)."""
    global _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
        return lib


def lib():
    return load()


def last_error() -> str:
    msg = lib().glm_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = ""):
    """Raise the reference's exception type for a non-zero status."""
    if status == GLM_OK:
        return
    from .solver import SolverDivergence, SolverError  # noqa: WPS433 (import cycle)
    msg = last_error() or what
    if status == GLM_SOLVER_ERROR:
        raise SolverError(msg)
    if status == GLM_DIVERGENCE:
        raise SolverDivergence(msg)
    if status == GLM_USAGE:
        raise ValueError(msg)
    raise GlmCudaError(f"{what}: {msg}")
