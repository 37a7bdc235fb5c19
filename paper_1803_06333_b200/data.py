"""Data layer: host containers with the reference's API plus their HBM twins.

Reference: data.py:42-464 (SparseColumnMatrix, parse_svmlight, partitions,
GLMCHUNK store). The host classes keep the reference's constructor, fields,
dtypes and error messages; every arithmetic method (col_sqnorms, matvec,
rmatvec, select/scale/transpose) runs on the GPU through the device twin
`DeviceMatrix`, whose index arrays are bit-identical to the reference's.

HBM layout: CSC = indptr i64[n+1], rows i32[nnz],
vals f64[nnz], sqnorms f64[n]; dense = column-major f64[d*n]. A contiguous
partition of columns is a zero-copy view (indptr offset, shared rows/vals).
"""

from __future__ import annotations

import ctypes
import os
import unicodedata
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

CHUNK_MAGIC = b"GLMCHUNK"
CHUNK_VERSION = 1
ENDIAN_MARK = 0xFEFF
_FLAG_LABELS = 1
_FLAG_ROW_VECTOR = 2


class DataFormatError(ValueError):
    """Malformed svmlight input."""


class ChunkFormatError(ValueError):
    """Corrupt or incompatible chunk file."""


class PartitionError(ValueError):
    """Requested partitioning is impossible."""


def _D():
    from . import _device
    return _device


# ---------------------------------------------------------------------------
class DeviceMatrix:
    """A matrix resident in HBM (CSC or dense column-major) + its glm_matrix view."""

    def __init__(self, n_rows, n_cols, layout, vals, indptr=None, rows=None, sqnorms=None,
                 labels=None, nnz=None, indptr_offset=0, keepalive=()):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.layout = layout
        self.vals = vals
        self.indptr = indptr
        self.rows = rows
        self.labels = labels
        self._keep = keepalive
        if nnz is None:
            nnz = self.n_rows * self.n_cols if layout == L.DENSE else int(indptr[-1].item())
        self.nnz = int(nnz)
        self.struct = L.GlmMatrix()
        self.struct.n_rows = self.n_rows
        self.struct.n_cols = self.n_cols
        self.struct.nnz = self.nnz
        self.struct.layout = layout
        self.struct.indptr = indptr.data_ptr() + 8 * indptr_offset if indptr is not None else None
        self.struct.rows = rows.data_ptr() if rows is not None else None
        self.struct.vals = vals.data_ptr()
        self._indptr_offset = indptr_offset
        self.sqnorms = sqnorms
        if sqnorms is None:
            self.sqnorms = torch.empty(max(self.n_cols, 1), dtype=torch.float64,
                                       device=vals.device)
            self.struct.sqnorms = self.sqnorms.data_ptr()
            if self.n_cols:
                L.check(L.lib().glm_col_sqnorms(ctypes.byref(self.struct),
                                                _D().ptr(self.sqnorms), _D().sptr()),
                        "glm_col_sqnorms")
        else:
            self.struct.sqnorms = sqnorms.data_ptr()

    # -- construction ------------------------------------------------------
    @classmethod
    def from_csc(cls, n_rows, indptr, rows, vals, labels=None, validate=False):
        D = _D()
        ip = D.to_device(indptr, torch.int64)
        rw = D.to_device(rows if len(rows) else np.zeros(1, np.int32), torch.int32)
        vl = D.to_device(vals if len(vals) else np.zeros(1), torch.float64)
        lab = D.to_device(labels) if labels is not None else None
        dm = cls(n_rows, len(indptr) - 1, L.CSC, vl, ip, rw, labels=lab, nnz=int(indptr[-1]))
        if validate:
            L.check(L.lib().glm_validate(ctypes.byref(dm.struct), D.sptr()), "glm_validate")
        return dm

    @classmethod
    def from_dense(cls, dense, labels=None):
        """dense: (n_rows, n_cols) array; stored column-major (column j contiguous)."""
        D = _D()
        arr = np.asarray(dense, dtype=np.float64)
        cm = np.ascontiguousarray(arr.T).reshape(-1)
        vl = D.to_device(cm)
        lab = D.to_device(labels) if labels is not None else None
        return cls(arr.shape[0], arr.shape[1], L.DENSE, vl, labels=lab)

    def columns(self, lo, hi):
        """Zero-copy view of columns [lo, hi) (a contiguous partition)."""
        lo, hi = int(lo), int(hi)
        sq = self.sqnorms[lo:hi] if hi > lo else self.sqnorms[:1]
        if self.layout == L.DENSE:
            v = self.vals[lo * self.n_rows:hi * self.n_rows] if hi > lo else self.vals[:1]
            return DeviceMatrix(self.n_rows, hi - lo, L.DENSE, v, sqnorms=sq,
                                labels=None if self.labels is None else self.labels[lo:hi],
                                keepalive=(self,))
        off = self._indptr_offset + lo
        nnz = int(self.indptr[off + (hi - lo)].item() - self.indptr[off].item())
        return DeviceMatrix(self.n_rows, hi - lo, L.CSC, self.vals, self.indptr, self.rows,
                            sqnorms=sq, nnz=nnz, indptr_offset=off,
                            labels=None if self.labels is None else self.labels[lo:hi],
                            keepalive=(self,))

    # -- arithmetic ----------------------------------------------------------
    def col_sqnorms(self):
        return self.sqnorms[:self.n_cols]

    def matvec(self, x, out=None, stream=None):
        D = _D()
        xd = D.to_device(x)
        out = out if out is not None else torch.empty(max(self.n_rows, 1), dtype=torch.float64,
                                                      device=xd.device)
        L.check(L.lib().glm_matvec(ctypes.byref(self.struct), D.ptr(xd), D.ptr(out),
                                   D.sptr(stream)), "glm_matvec")
        return out[:self.n_rows]

    def rmatvec(self, w, out=None, stream=None):
        D = _D()
        wd = D.to_device(w)
        out = out if out is not None else torch.empty(max(self.n_cols, 1), dtype=torch.float64,
                                                      device=wd.device)
        if self.n_cols:
            L.check(L.lib().glm_rmatvec(ctypes.byref(self.struct), D.ptr(wd), D.ptr(out),
                                        D.sptr(stream)), "glm_rmatvec")
        return out[:self.n_cols]

    def _csc_arrays(self):
        off = self._indptr_offset
        ip = self.indptr[off:off + self.n_cols + 1]
        base = int(ip[0].item())
        return ip - base, self.rows[base:base + self.nnz], self.vals[base:base + self.nnz]

    def transpose(self):
        """Stable transpose (data.py:155-165) on the GPU; labels dropped."""
        if self.layout == L.DENSE:
            return DeviceMatrix.from_dense(self.to_dense_numpy().T)
        D = _D()
        if self._indptr_offset == 0 and int(self.indptr[0].item()) == 0:
            src = self
        else:
            ip, rw, vl = self._csc_arrays()
            src = DeviceMatrix(self.n_rows, self.n_cols, L.CSC, vl.contiguous(), ip.contiguous(),
                               rw.contiguous(), sqnorms=self.sqnorms, nnz=self.nnz)
        dev = self.vals.device
        ip_t = torch.empty(self.n_rows + 1, dtype=torch.int64, device=dev)
        rows_t = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
        vals_t = torch.empty(max(self.nnz, 1), dtype=torch.float64, device=dev)
        nb = L.lib().glm_transpose_temp_bytes(self.nnz, self.n_rows)
        tmp = torch.empty(nb, dtype=torch.uint8, device=dev)
        L.check(L.lib().glm_transpose(ctypes.byref(src.struct), D.ptr(ip_t), D.ptr(rows_t),
                                      D.ptr(vals_t), D.ptr(tmp), nb, D.sptr()), "glm_transpose")
        return DeviceMatrix(self.n_cols, self.n_rows, L.CSC, vals_t, ip_t, rows_t, nnz=self.nnz)

    def select_columns(self, cols):
        """Copy of the given columns (data.py:132-145), gathered on the GPU."""
        D = _D()
        cols_d = D.to_device(np.asarray(cols, dtype=np.int64), torch.int64)
        k = int(cols_d.numel())
        dev = self.vals.device
        if self.layout == L.DENSE:
            idx = cols_d
            mat = self.vals[:self.n_rows * self.n_cols].view(self.n_cols, self.n_rows)
            vals = mat.index_select(0, idx).reshape(-1).contiguous() if k else \
                torch.zeros(1, dtype=torch.float64, device=dev)
            lab = self.labels.index_select(0, idx) if self.labels is not None and k else None
            return DeviceMatrix(self.n_rows, k, L.DENSE, vals, labels=lab)
        ip = torch.empty(k + 1, dtype=torch.int64, device=dev)
        nb = L.lib().glm_select_temp_bytes(k)
        tmp = torch.empty(nb, dtype=torch.uint8, device=dev)
        L.check(L.lib().glm_select_indptr(ctypes.byref(self.struct), D.ptr(cols_d), k, D.ptr(ip),
                                          D.ptr(tmp), nb, D.sptr()), "glm_select_indptr")
        nnz = int(ip[-1].item())
        rows = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        L.check(L.lib().glm_select_gather(ctypes.byref(self.struct), D.ptr(cols_d), k, D.ptr(ip),
                                          D.ptr(rows), D.ptr(vals), D.sptr()),
                "glm_select_gather")
        lab = self.labels.index_select(0, cols_d) if self.labels is not None and k else None
        return DeviceMatrix(self.n_rows, k, L.CSC, vals, ip, rows, labels=lab, nnz=nnz)

    def scale_columns(self, scales):
        """New matrix with column j multiplied by scales[j] (data.py:147-153)."""
        D = _D()
        sc = D.to_device(scales)
        out = torch.empty_like(self.vals)
        L.check(L.lib().glm_scale_columns(ctypes.byref(self.struct), D.ptr(sc), D.ptr(out),
                                          D.sptr()), "glm_scale_columns")
        if self.layout == L.DENSE:
            return DeviceMatrix(self.n_rows, self.n_cols, L.DENSE, out, labels=self.labels)
        return DeviceMatrix(self.n_rows, self.n_cols, L.CSC, out, self.indptr, self.rows,
                            labels=self.labels, nnz=self.nnz, indptr_offset=self._indptr_offset)

    # -- host views ----------------------------------------------------------
    def to_dense_numpy(self):
        if self.layout == L.DENSE:
            return _D().to_host(self.vals[:self.n_rows * self.n_cols]).reshape(
                self.n_cols, self.n_rows).T.copy()
        return self.to_host().to_dense()

    def to_host(self):
        D = _D()
        if self.layout == L.DENSE:
            dense = self.to_dense_numpy()
            rows, cols = np.nonzero(dense.T)
            indptr = np.searchsorted(rows, np.arange(self.n_cols + 1))
            return SparseColumnMatrix(self.n_rows, indptr, cols, dense.T[rows, cols],
                                      validate=False)
        ip, rw, vl = self._csc_arrays()
        lab = D.to_host(self.labels) if self.labels is not None else None
        return SparseColumnMatrix(self.n_rows, D.to_host(ip), D.to_host(rw)[:self.nnz],
                                  D.to_host(vl)[:self.nnz], lab, validate=False)


# ---------------------------------------------------------------------------
class SparseColumnMatrix:
    """Immutable CSC-like sparse matrix with optional per-column labels
    (data.py:42-171). Host container; arithmetic runs on its DeviceMatrix."""

    __slots__ = ("n_rows", "n_cols", "indptr", "rows", "vals", "labels", "_sqnorms", "_dev")

    def __init__(self, n_rows, indptr, rows, vals, labels=None, validate=True):
        self.n_rows = int(n_rows)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.rows = np.ascontiguousarray(rows, dtype=np.int32)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.n_cols = len(self.indptr) - 1
        if labels is not None:
            labels = np.ascontiguousarray(labels, dtype=np.float64)
        self.labels = labels
        self._sqnorms = None
        self._dev = None
        if validate:
            self._validate()

    def _validate(self):
        """The reference's input checks, in its order, with its messages
        (data.py:64-84)."""
        ip, rw, vl = self.indptr, self.rows, self.vals
        nnz = len(rw)
        checks = (
            (lambda: ip[0] == 0 and ip[-1] == nnz, "indptr does not span the value arrays"),
            (lambda: bool(np.all(ip[1:] >= ip[:-1])), "indptr must be non-decreasing"),
            (lambda: len(vl) == nnz, "rows/vals length mismatch"),
            (lambda: nnz == 0 or (int(rw.min()) >= 0 and int(rw.max()) < self.n_rows),
             "row index out of range"),
            (lambda: nnz == 0 or bool(np.isfinite(vl).all()), "non-finite value in matrix"),
            (self._rows_increase, "row indices must be strictly increasing per column"),
            (lambda: self.labels is None or len(self.labels) == self.n_cols,
             "labels length must equal n_cols"),
        )
        for holds, message in checks:
            if not holds():
                raise ValueError(message)

    def _rows_increase(self):
        """An entry may sit at or below its predecessor only where a column
        starts (sorted, unique rows per column)."""
        if len(self.rows) < 2:
            return True
        drops = np.flatnonzero(self.rows[1:] <= self.rows[:-1]) + 1
        return bool(np.isin(drops, self.indptr).all())

    @property
    def nnz(self):
        return int(self.indptr[-1])

    def device(self) -> DeviceMatrix:
        """The HBM twin (uploaded once, cached)."""
        if self._dev is None:
            self._dev = DeviceMatrix.from_csc(self.n_rows, self.indptr, self.rows, self.vals,
                                              self.labels)
        return self._dev

    def col(self, j):
        lo, hi = self.indptr[j], self.indptr[j + 1]
        return self.rows[lo:hi], self.vals[lo:hi]

    def col_nnz(self):
        return np.diff(self.indptr)

    def col_sqnorms(self):
        if self._sqnorms is None:
            self._sqnorms = _D().to_host(self.device().col_sqnorms()).copy()
        return self._sqnorms

    def matvec(self, x):
        return _D().to_host(self.device().matvec(x)).copy()

    def rmatvec(self, w):
        return _D().to_host(self.device().rmatvec(w)).copy()

    def to_dense(self):
        out = np.zeros((self.n_rows, self.n_cols))
        cols = np.repeat(np.arange(self.n_cols), np.diff(self.indptr))
        out[self.rows, cols] = self.vals
        return out

    def select_columns(self, cols):
        return self.device().select_columns(cols).to_host()

    def scale_columns(self, scales):
        out = self.device().scale_columns(scales).to_host()
        out.labels = None if self.labels is None else self.labels.copy()
        return out

    def transpose(self):
        return self.device().transpose().to_host()

    def value_equal(self, other):
        return (self.n_rows == other.n_rows and self.n_cols == other.n_cols
                and np.array_equal(self.indptr, other.indptr)
                and np.array_equal(self.rows, other.rows)
                and np.array_equal(self.vals, other.vals))


class DenseColumnMatrix:
    """Dense (n_rows, n_cols) design stored column-major in HBM (C1/C3 shapes)."""

    def __init__(self, dense, labels=None):
        self.dense = np.asarray(dense, dtype=np.float64)
        self.n_rows, self.n_cols = self.dense.shape
        self.labels = None if labels is None else np.asarray(labels, dtype=np.float64)
        self._dev = None

    @property
    def nnz(self):
        return self.n_rows * self.n_cols

    def device(self) -> DeviceMatrix:
        if self._dev is None:
            self._dev = DeviceMatrix.from_dense(self.dense, self.labels)
        return self._dev

    def col_nnz(self):
        return np.full(self.n_cols, self.n_rows, dtype=np.int64)

    def col_sqnorms(self):
        return _D().to_host(self.device().col_sqnorms()).copy()

    def matvec(self, x):
        return _D().to_host(self.device().matvec(x)).copy()

    def rmatvec(self, w):
        return _D().to_host(self.device().rmatvec(w)).copy()

    def to_dense(self):
        return self.dense.copy()


def hstack(blocks):
    """Column-wise concatenation (data.py:174-187): each block's indptr is
    shifted by the entries before it; labels survive only if every block
    has them."""
    blocks = list(blocks)
    n_rows = blocks[0].n_rows
    if any(b.n_rows != n_rows for b in blocks):
        raise ValueError("n_rows mismatch in hstack")
    shift = np.cumsum([0] + [int(b.indptr[-1] - b.indptr[0]) for b in blocks[:-1]],
                      dtype=np.int64)
    indptr = np.concatenate([np.zeros(1, np.int64)] +
                            [np.asarray(b.indptr[1:], np.int64) - b.indptr[0] + o
                             for b, o in zip(blocks, shift)])
    rows = np.concatenate([b.rows for b in blocks])
    vals = np.concatenate([b.vals for b in blocks])
    has_labels = all(b.labels is not None for b in blocks)
    labels = np.concatenate([b.labels for b in blocks]) if has_labels else None
    return SparseColumnMatrix(n_rows, indptr, rows, vals, labels, validate=False)


# --------------------------------------------------------------- svmlight
# Characters outside the native parser's ASCII grammar whose meaning Python's
# str.split/strip/float give them: every whitespace character separates, and
# int()/float() read any Unicode decimal digit (CPython maps both to ASCII
# before parsing a number); anything else is just an invalid character.
_EXOTIC_ASCII = "\x1c\x1d\x1e\x1f"


def _to_grammar(text):
    """Map `text` one character to one ASCII character so the native grammar
    sees what Python's line parsing would: offsets into the result are
    offsets into `text` (error tokens are cut from the original)."""
    if text.isascii() and not any(c in text for c in _EXOTIC_ASCII):
        return text
    table = {}
    for ch in set(text):
        if ch == "\n" or (ch.isascii() and ch not in _EXOTIC_ASCII):
            continue
        if ch.isspace():
            table[ord(ch)] = " "
        else:
            dig = unicodedata.decimal(ch, None)
            table[ord(ch)] = str(dig) if dig is not None else "\x01"
    return text.translate(table)


def parse_svmlight(stream, n_threads=0):
    """svmlight text -> (example-major matrix, labels) (data.py:190-239).

    Host ingest by the multi-threaded native parser
    (csrc/ingest.cu, `glm_svmlight_parse`).  The input is first brought to
    the lines the reference iterates: a str is cut with str.splitlines(), a
    file object at its newlines, an iterable gives one line per item; the
    native error report (kind, line, token offsets) becomes the reference's
    exception and message here."""
    if isinstance(stream, str):
        text = "\n".join(stream.splitlines())
    elif hasattr(stream, "read"):
        text = stream.read()
        if isinstance(text, bytes):
            text = text.decode()
    else:
        text = "\n".join((ln.decode() if isinstance(ln, bytes) else ln).replace("\n", " ")
                         for ln in stream)
    data = _to_grammar(text).encode("ascii")
    lib = L.lib()
    h = ctypes.c_void_p()
    info = np.zeros(7, dtype=np.int64)
    L.check(lib.glm_svmlight_parse(data, len(data), int(n_threads), ctypes.byref(h),
                                   info.ctypes.data_as(ctypes.c_void_p)), "glm_svmlight_parse")
    if info[3] != 0:
        _raise_parse_error(int(info[3]), int(info[4]), text[info[5]:info[5] + info[6]])
    n, nnz, max_feat = int(info[0]), int(info[1]), int(info[2])
    arrays = (np.empty(n + 1, np.int64), np.empty(nnz, np.int32), np.empty(nnz, np.float64),
              np.empty(n, np.float64))
    try:
        L.check(lib.glm_svmlight_fetch(h, *(a.ctypes.data_as(ctypes.c_void_p) for a in arrays)),
                "glm_svmlight_fetch")
    finally:
        lib.glm_svmlight_free(h)
    indptr, rows, vals, labels = arrays
    return SparseColumnMatrix(max_feat, indptr, rows, vals), labels


def _raise_parse_error(kind, line, token):
    """The reference's exception for the native parser's first error."""
    where = f"line {line}: "
    if kind == 1:
        raise DataFormatError(where + f"bad label {token!r}")
    if kind == 2:
        raise DataFormatError(where + f"bad feature token {token!r}")
    if kind == 3:
        raise DataFormatError(where + f"feature index {int(token.split(':', 1)[0])} < 1")
    if kind == 4:
        raise DataFormatError(where + "feature indices must be strictly increasing")
    # kind 5: an index past int32 — the reference fails converting its row
    # list (np.asarray(rows, dtype=np.int32)); let numpy raise the same error
    np.asarray([int(token.split(":", 1)[0]) - 1], dtype=np.int32)
    raise OverflowError(f"feature index out of int32 range at line {line}")


def write_svmlight(matrix, labels, stream):
    """Example-major matrix -> svmlight text (data.py:242-250): every number
    as %.17g, so parsing the text returns the same bits."""
    tokens = [f"{r + 1}:{v:.17g}" for r, v in zip(matrix.rows.tolist(), matrix.vals.tolist())]
    ends = np.asarray(matrix.indptr).tolist()
    for j, y in enumerate(np.asarray(labels, dtype=np.float64).tolist()):
        stream.write(" ".join([f"{y:.17g}"] + tokens[ends[j]:ends[j + 1]]) + "\n")


# -------------------------------------------------------------- partitions
@dataclass(frozen=True)
class Partition:
    node: int
    device: int
    cols: np.ndarray

    def __len__(self):
        return len(self.cols)

    @property
    def lo(self):
        return int(self.cols[0]) if len(self.cols) else 0

    @property
    def hi(self):
        return int(self.cols[-1]) + 1 if len(self.cols) else 0


def partition_bounds(n_cols, n_nodes, n_devices, strategy="contiguous", col_nnz=None):
    """Worker boundaries of partition_columns (data.py:264-304): W+1 ints."""
    if n_nodes < 1 or n_devices < 1 or n_cols < 1:
        raise PartitionError("need n_cols, nodes and devices all >= 1")
    workers = n_nodes * n_devices
    if workers > n_cols:
        raise PartitionError(f"{workers} workers but only {n_cols} coordinates to assign")
    if strategy == "contiguous":
        q, r = divmod(n_cols, workers)   # np.array_split: first r parts get +1
        sizes = [q + 1] * r + [q] * (workers - r)
        return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    if strategy == "balanced-by-nnz":
        if col_nnz is None:
            raise PartitionError("balanced-by-nnz requires col_nnz")
        csum = np.cumsum(np.asarray(col_nnz, dtype=np.int64))
        total = csum[-1] if n_cols else 0
        bounds = [0]
        for m in range(1, workers):
            b = int(np.searchsorted(csum, total * m / workers))
            b = max(b, bounds[-1] + 1)
            b = min(b, n_cols - (workers - m))
            bounds.append(b)
        bounds.append(n_cols)
        return np.array(bounds, dtype=np.int64)
    raise PartitionError(f"unknown strategy {strategy!r}")


def partition_columns(n_cols, n_nodes, n_devices, strategy="contiguous", col_nnz=None):
    """K*L disjoint sorted contiguous coordinate sets (data.py:264-288)."""
    b = partition_bounds(n_cols, n_nodes, n_devices, strategy, col_nnz)
    return [Partition(node=w // n_devices, device=w % n_devices,
                      cols=np.arange(b[w], b[w + 1], dtype=np.int64))
            for w in range(n_nodes * n_devices)]


# ----------------------------------------------------------- chunk store
@dataclass
class ChunkDescriptor:
    offset: int
    n_cols: int
    nnz: int


@dataclass
class ChunkStore:
    path: str
    n_rows: int
    n_cols: int
    has_labels: bool
    chunks: list = field(default_factory=list)
    row_vector: np.ndarray | None = None

    @property
    def n_chunks(self):
        return len(self.chunks)


_CHUNK_ERRORS = {1: "truncated header", 3: "endianness mismatch", 5: "truncated row vector",
                 6: "truncated chunk header", 7: "chunk column counts do not sum to n_cols",
                 8: "chunk header disagrees with descriptor", 9: "truncated chunk body"}


def _chunk_error(kind, path, errno_=0, magic=b"", version=0):
    if kind == 10:
        raise OSError(errno_, os.strerror(errno_), str(path))
    if kind == 2:
        raise ChunkFormatError(f"bad magic {magic!r}")
    if kind == 4:
        raise ChunkFormatError(f"unsupported version {version}")
    raise ChunkFormatError(_CHUNK_ERRORS[kind])


def write_chunks(matrix, chunk_size, path, row_vector=None):
    """GLMCHUNK v1 writer (data.py:329-359) — native (csrc/chunkfile.cu),
    byte-identical to the reference's files."""
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    if row_vector is not None:
        row_vector = np.ascontiguousarray(row_vector, dtype=np.float64)
        if len(row_vector) != matrix.n_rows:
            raise ValueError("row_vector length must equal n_rows")
    labels = None if matrix.labels is None else np.ascontiguousarray(matrix.labels, np.float64)
    n_chunks = -(-matrix.n_cols // chunk_size)
    offsets = np.zeros(max(n_chunks, 1), np.int64)
    err = ctypes.c_int64(0)
    vp = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    L.check(L.lib().glm_chunk_write(os.fsencode(path), matrix.n_rows, matrix.n_cols,
                                    vp(matrix.indptr), vp(matrix.rows), vp(matrix.vals),
                                    vp(labels), vp(row_vector), int(chunk_size), vp(offsets),
                                    ctypes.byref(err)), "glm_chunk_write")
    if err.value:
        _chunk_error(10, path, err.value)
    sizes = np.diff(np.minimum(np.arange(n_chunks + 1) * chunk_size, matrix.n_cols))
    nnz = np.diff(matrix.indptr[np.minimum(np.arange(n_chunks + 1) * chunk_size, matrix.n_cols)])
    store = ChunkStore(path=path, n_rows=matrix.n_rows, n_cols=matrix.n_cols,
                       has_labels=labels is not None, row_vector=row_vector)
    store.chunks = [ChunkDescriptor(int(o), int(c), int(z))
                    for o, c, z in zip(offsets[:n_chunks], sizes, nnz)]
    return store


def open_chunks(path):
    """Scan a chunk file into its descriptor table (data.py:362-398), natively."""
    lib = L.lib()
    h = ctypes.c_void_p()
    info = np.zeros(8, np.int64)
    magic = ctypes.create_string_buffer(8)
    L.check(lib.glm_chunk_open(os.fsencode(path), ctypes.byref(h),
                               info.ctypes.data_as(ctypes.c_void_p), magic), "glm_chunk_open")
    if info[0]:
        _chunk_error(int(info[0]), path, int(info[6]), magic.raw, int(info[4]))
    n_rows, n_cols, flags, k = int(info[1]), int(info[2]), int(info[3]), int(info[5])
    table = np.zeros((3, max(k, 1)), np.int64)
    rv = np.zeros(n_rows, np.float64) if flags & _FLAG_ROW_VECTOR else None
    try:
        L.check(lib.glm_chunk_table(h, *(table[i].ctypes.data_as(ctypes.c_void_p)
                                         for i in range(3)),
                                    None if rv is None else rv.ctypes.data_as(ctypes.c_void_p)),
                "glm_chunk_table")
    finally:
        lib.glm_chunk_close(h)
    store = ChunkStore(path=path, n_rows=n_rows, n_cols=n_cols,
                       has_labels=bool(flags & _FLAG_LABELS), row_vector=rv)
    store.chunks = [ChunkDescriptor(int(o), int(c), int(z)) for o, c, z in table[:, :k].T]
    return store


def read_chunk(store, index):
    """Chunk `index` as a SparseColumnMatrix (data.py:401-426), read natively;
    the on-disk u64/u32 arrays are the same bits as i64/i32."""
    desc = store.chunks[index]
    c, z = desc.n_cols, desc.nnz
    indptr, rows, vals = np.empty(c + 1, np.int64), np.empty(z, np.int32), np.empty(z, np.float64)
    labels = np.empty(c, np.float64) if store.has_labels else None
    status = np.zeros(2, np.int64)
    vp = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    L.check(L.lib().glm_chunk_read(os.fsencode(store.path), desc.offset, c, z,
                                   int(store.has_labels), vp(indptr), vp(rows), vp(vals),
                                   vp(labels), vp(status)), "glm_chunk_read")
    if status[0]:
        _chunk_error(int(status[0]), store.path, int(status[1]))
    return SparseColumnMatrix(store.n_rows, indptr, rows, vals, labels, validate=False)


def concat_chunks(store):
    return hstack(read_chunk(store, i) for i in range(store.n_chunks))
