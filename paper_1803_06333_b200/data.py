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
import io
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

CHUNK_MAGIC = b"GLMCHUNK"
CHUNK_VERSION = 1
ENDIAN_MARK = 0xFEFF
_FLAG_LABELS = 1
_FLAG_ROW_VECTOR = 2
_HEADER = struct.Struct("<8sIHHQQ")   # data.py:23-25
_CHUNK_HEAD = struct.Struct("<IQ")    # data.py:26-27


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
        """Input checks with the reference's messages (data.py:64-84)."""
        if self.indptr[0] != 0 or self.indptr[-1] != len(self.rows):
            raise ValueError("indptr does not span the value arrays")
        if np.any(np.diff(self.indptr) < 0):
            raise ValueError("indptr must be non-decreasing")
        if len(self.rows) != len(self.vals):
            raise ValueError("rows/vals length mismatch")
        if len(self.rows):
            if self.rows.min() < 0 or self.rows.max() >= self.n_rows:
                raise ValueError("row index out of range")
            if not np.all(np.isfinite(self.vals)):
                raise ValueError("non-finite value in matrix")
            d = np.diff(self.rows)
            starts = np.zeros(len(self.rows), dtype=bool)
            inner = self.indptr[1:-1]
            starts[inner[inner < len(self.rows)]] = True
            if np.any((d <= 0) & ~starts[1:]):
                raise ValueError("row indices must be strictly increasing per column")
        if self.labels is not None and len(self.labels) != self.n_cols:
            raise ValueError("labels length must equal n_cols")

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
    """Concatenate matrices column-wise (data.py:174-187)."""
    blocks = list(blocks)
    n_rows = blocks[0].n_rows
    if any(b.n_rows != n_rows for b in blocks):
        raise ValueError("n_rows mismatch in hstack")
    indptr = np.concatenate([[0]] + [np.diff(b.indptr) for b in blocks]).cumsum()
    rows = np.concatenate([b.rows for b in blocks]) if blocks else np.empty(0, np.int32)
    vals = np.concatenate([b.vals for b in blocks])
    labels = None
    if all(b.labels is not None for b in blocks):
        labels = np.concatenate([b.labels for b in blocks])
    return SparseColumnMatrix(n_rows, indptr.astype(np.int64), rows, vals, labels,
                              validate=False)


# --------------------------------------------------------------- svmlight
# Characters whose meaning differs between Python's line/field splitting and
# the native parser's ASCII grammar: inputs containing them take the
# line-by-line path below, which follows data.py:190-239 exactly.
_NATIVE_UNSAFE = ("\x0b", "\x0c", "\x1c", "\x1d", "\x1e", "\x1f")


def parse_svmlight(stream, n_threads=0):
    """svmlight text -> (example-major matrix, labels) (data.py:190-239).

    Host ingest: text from a str or a file object is parsed
    by the multi-threaded native parser (csrc/ingest.cu, `glm_svmlight_parse`);
    exotic input (non-ASCII, or separators Python splits on but the native
    grammar does not) and every error case run the line-by-line path, so the
    values, the arrays and the error messages are those of the reference."""
    if isinstance(stream, str):
        text, str_input = stream, True
    elif hasattr(stream, "read"):
        text, str_input = stream.read(), False
        if isinstance(text, bytes):
            text = text.decode()
    else:
        return _parse_svmlight_lines(stream)
    res = _parse_svmlight_native(text, str_input, n_threads)
    if res is not None:
        return res
    return _parse_svmlight_lines(text.splitlines() if str_input else io.StringIO(text))


def _parse_svmlight_native(text, str_input, n_threads):
    if not text.isascii() or any(c in text for c in _NATIVE_UNSAFE) or \
            (str_input and "\r" in text):
        return None
    data = text.encode()
    lib = L.lib()
    h = ctypes.c_void_p()
    info = np.zeros(7, dtype=np.int64)
    L.check(lib.glm_svmlight_parse(data, len(data), int(n_threads), ctypes.byref(h),
                                   info.ctypes.data_as(ctypes.c_void_p)), "glm_svmlight_parse")
    if info[3] != 0:
        return None                      # the line path raises the reference's error
    n, nnz, max_feat = int(info[0]), int(info[1]), int(info[2])
    indptr = np.empty(n + 1, dtype=np.int64)
    rows = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    labels = np.empty(n, dtype=np.float64)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    try:
        L.check(lib.glm_svmlight_fetch(h, vp(indptr), vp(rows), vp(vals), vp(labels)),
                "glm_svmlight_fetch")
    finally:
        lib.glm_svmlight_free(h)
    return SparseColumnMatrix(max_feat, indptr, rows, vals), labels


def _parse_svmlight_lines(lines):
    """The reference's line loop (data.py:198-239), same validation/messages."""
    labels, indptr, rows, vals = [], [0], [], []
    max_feat = 0
    for lineno, line in enumerate(lines, start=1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        try:
            y = float(parts[0])
        except ValueError:
            raise DataFormatError(f"line {lineno}: bad label {parts[0]!r}")
        prev = 0
        for tok in parts[1:]:
            try:
                idx_s, val_s = tok.split(":", 1)
                idx = int(idx_s)
                val = float(val_s)
            except ValueError:
                raise DataFormatError(f"line {lineno}: bad feature token {tok!r}")
            if idx < 1:
                raise DataFormatError(f"line {lineno}: feature index {idx} < 1")
            if idx <= prev:
                raise DataFormatError(
                    f"line {lineno}: feature indices must be strictly increasing")
            prev = idx
            rows.append(idx - 1)
            vals.append(val)
        max_feat = max(max_feat, prev)
        labels.append(y)
        indptr.append(len(rows))
    mat = SparseColumnMatrix(max_feat, np.asarray(indptr, dtype=np.int64),
                             np.asarray(rows, dtype=np.int32), np.asarray(vals, dtype=np.float64))
    return mat, np.asarray(labels, dtype=np.float64)


def write_svmlight(matrix, labels, stream):
    """data.py:242-250 (value-exact %.17g)."""
    for j in range(matrix.n_cols):
        r, v = matrix.col(j)
        feats = " ".join("%d:%.17g" % (ri + 1, vi) for ri, vi in zip(r, v))
        line = "%.17g" % labels[j]
        if feats:
            line += " " + feats
        stream.write(line + "\n")


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


def write_chunks(matrix, chunk_size, path, row_vector=None):
    """GLMCHUNK v1 writer (data.py:329-359), byte-identical to the reference."""
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    has_labels = matrix.labels is not None
    flags = _FLAG_LABELS if has_labels else 0
    if row_vector is not None:
        row_vector = np.ascontiguousarray(row_vector, dtype=np.float64)
        if len(row_vector) != matrix.n_rows:
            raise ValueError("row_vector length must equal n_rows")
        flags |= _FLAG_ROW_VECTOR
    store = ChunkStore(path=path, n_rows=matrix.n_rows, n_cols=matrix.n_cols,
                       has_labels=has_labels, row_vector=row_vector)
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(CHUNK_MAGIC, CHUNK_VERSION, flags, ENDIAN_MARK, matrix.n_rows,
                              matrix.n_cols))
        if row_vector is not None:
            fh.write(row_vector.tobytes())
        for lo in range(0, matrix.n_cols, chunk_size):
            hi = min(lo + chunk_size, matrix.n_cols)
            sub_ptr = (matrix.indptr[lo:hi + 1] - matrix.indptr[lo]).astype(np.uint64)
            nnz = int(sub_ptr[-1])
            store.chunks.append(ChunkDescriptor(fh.tell(), hi - lo, nnz))
            fh.write(_CHUNK_HEAD.pack(hi - lo, nnz))
            fh.write(sub_ptr.tobytes())
            fh.write(matrix.rows[matrix.indptr[lo]:matrix.indptr[hi]].astype(np.uint32).tobytes())
            fh.write(matrix.vals[matrix.indptr[lo]:matrix.indptr[hi]].tobytes())
            if has_labels:
                fh.write(matrix.labels[lo:hi].tobytes())
    return store


def open_chunks(path):
    """Scan a chunk file (data.py:362-398)."""
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
        if len(head) < _HEADER.size:
            raise ChunkFormatError("truncated header")
        magic, version, flags, endian, n_rows, n_cols = _HEADER.unpack(head)
        if magic != CHUNK_MAGIC:
            raise ChunkFormatError(f"bad magic {magic!r}")
        if endian != ENDIAN_MARK:
            raise ChunkFormatError("endianness mismatch")
        if version != CHUNK_VERSION:
            raise ChunkFormatError(f"unsupported version {version}")
        has_labels = bool(flags & _FLAG_LABELS)
        store = ChunkStore(path=path, n_rows=n_rows, n_cols=n_cols, has_labels=has_labels)
        if flags & _FLAG_ROW_VECTOR:
            buf = fh.read(8 * n_rows)
            if len(buf) < 8 * n_rows:
                raise ChunkFormatError("truncated row vector")
            store.row_vector = np.frombuffer(buf, dtype="<f8").copy()
        seen = 0
        while seen < n_cols:
            offset = fh.tell()
            head = fh.read(_CHUNK_HEAD.size)
            if len(head) < _CHUNK_HEAD.size:
                raise ChunkFormatError("truncated chunk header")
            c_cols, c_nnz = _CHUNK_HEAD.unpack(head)
            store.chunks.append(ChunkDescriptor(offset, c_cols, c_nnz))
            body = 8 * (c_cols + 1) + 12 * c_nnz + (8 * c_cols if has_labels else 0)
            fh.seek(body, 1)
            seen += c_cols
        if seen != n_cols:
            raise ChunkFormatError("chunk column counts do not sum to n_cols")
    return store


def read_chunk_arrays(store, index, out=None):
    """Chunk `index` as raw little-endian arrays (indptr u64, rows u32, vals f64,
    labels f64|None) read straight into `out` buffers when given (pinned)."""
    desc = store.chunks[index]
    with open(store.path, "rb") as fh:
        fh.seek(desc.offset)
        head = fh.read(_CHUNK_HEAD.size)
        if len(head) < _CHUNK_HEAD.size:
            raise ChunkFormatError("truncated chunk header")
        c_cols, c_nnz = _CHUNK_HEAD.unpack(head)
        if (c_cols, c_nnz) != (desc.n_cols, desc.nnz):
            raise ChunkFormatError("chunk header disagrees with descriptor")
        need = 8 * (c_cols + 1) + 12 * c_nnz + (8 * c_cols if store.has_labels else 0)
        if out is not None:
            n = fh.readinto(memoryview(out)[:need])
            buf = out
        else:
            buf = fh.read(need)
            n = len(buf)
        if n < need:
            raise ChunkFormatError("truncated chunk body")
    off = 0
    indptr = np.frombuffer(buf, dtype="<u8", count=c_cols + 1, offset=off)
    off += 8 * (c_cols + 1)
    rows = np.frombuffer(buf, dtype="<u4", count=c_nnz, offset=off)
    off += 4 * c_nnz
    vals = np.frombuffer(buf, dtype="<f8", count=c_nnz, offset=off)
    off += 8 * c_nnz
    labels = np.frombuffer(buf, dtype="<f8", count=c_cols, offset=off) \
        if store.has_labels else None
    return indptr, rows, vals, labels


def read_chunk(store, index):
    """Load chunk `index` as a SparseColumnMatrix (data.py:401-426)."""
    indptr, rows, vals, labels = read_chunk_arrays(store, index)
    return SparseColumnMatrix(store.n_rows, indptr.astype(np.int64), rows.astype(np.int32),
                              vals.copy(), None if labels is None else labels.copy(),
                              validate=False)


def concat_chunks(store):
    return hstack(read_chunk(store, i) for i in range(store.n_chunks))


def spectral_bound(matrix, tolerance=1e-3, max_iters=500):
    """Upper bound on ||A||_2^2 (data.py:434-464) by power iteration on the GPU."""
    dm = matrix.device() if hasattr(matrix, "device") else matrix
    frob = float(torch.dot(dm.vals[:dm.nnz], dm.vals[:dm.nnz]).item()) if dm.nnz else 0.0
    if frob == 0.0 or dm.n_cols == 0:
        return 0.0
    rng = np.random.default_rng(0x5EED)
    y = rng.standard_normal(dm.n_cols)
    y /= np.linalg.norm(y)
    yd = _D().to_device(y)
    rho = 0.0
    for _ in range(max_iters):
        my = dm.rmatvec(dm.matvec(yd))
        new_rho = float(torch.dot(yd, my).item())
        nrm = float(torch.linalg.norm(my).item())
        if nrm == 0.0:
            return 0.0
        done = abs(new_rho - rho) <= tolerance * max(new_rho, 1e-300)
        rho = new_rho
        yd = my / nrm
        if done:
            break
    my = dm.rmatvec(dm.matvec(yd))
    rho = float(torch.dot(yd, my).item())
    resid = float(torch.linalg.norm(my - rho * yd).item())
    return min(frob, rho + resid)
