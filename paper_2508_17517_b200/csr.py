"""Device CSR container and the sparse kernels of the AIRG path.

Mirrors the reference's ``airmg.sparse`` interface (sparse.py:18-30, 44-367):
``SparseMatrix``, ``validate``, ``spmv``, ``spgemm``, ``spgemm_fixed_sparsity``,
``extract``, ``drop_and_lump``, ``diagonal``.  Storage lives in HBM as
int32 row offsets / int32 columns / fp64 values (torch tensors used only as
device buffers); every operation is an sm_100a kernel in libairg.so.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

IDX = torch.int32
VAL = torch.float64


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError('paper_2508_17517_b200 needs a CUDA device (sm_100a); '
                           'there is no CPU fallback')
    return torch.device('cuda', torch.cuda.current_device())


def to_dev(a, dtype):
    """numpy / torch / list -> contiguous device tensor of ``dtype``."""
    if isinstance(a, torch.Tensor):
        return a.to(device=_dev(), dtype=dtype).contiguous()
    np_dtype = {IDX: np.int32, VAL: np.float64, torch.int8: np.int8,
                torch.int64: np.int64}[dtype]
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np_dtype)).to(_dev())


def empty(n, dtype):
    return torch.empty(max(int(n), 0), dtype=dtype, device=_dev())


@dataclass(frozen=True, eq=False)
class SparseMatrix:
    """Canonical CSR matrix resident in GPU memory (ref: sparse.py:44-152).

    ``row_offsets`` / ``col_indices`` are int32 device tensors, ``values`` fp64.
    """

    nrows: int
    ncols: int
    row_offsets: torch.Tensor
    col_indices: torch.Tensor
    values: torch.Tensor

    @classmethod
    def csr(cls, nrows, ncols, row_offsets, col_indices, values, check=True):
        A = cls(int(nrows), int(ncols), to_dev(row_offsets, IDX), to_dev(col_indices, IDX),
                to_dev(values, VAL))
        if check:
            validate(A)
        return A

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, values):
        """COO -> canonical CSR (host-side assembly utility, sparse.py:75-97)."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        values = np.asarray(values, dtype=np.float64)
        if not (len(rows) == len(cols) == len(values)):
            raise ValueError('coordinate arrays must have equal length')
        if len(rows) and (rows.min() < 0 or rows.max() >= nrows or cols.min() < 0
                          or cols.max() >= ncols):
            raise ValueError('coordinate entry out of range')
        o = np.lexsort((cols, rows))
        rows, cols, values = rows[o], cols[o], values[o]
        if len(rows):
            head = np.ones(len(rows), dtype=bool)
            head[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
            s = np.flatnonzero(head)
            values = np.add.reduceat(values, s)
            rows, cols = rows[s], cols[s]
        ptr = np.zeros(nrows + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=nrows), out=ptr[1:])
        return cls.csr(nrows, ncols, ptr, cols, values, check=False)

    @classmethod
    def from_dense(cls, arr):
        arr = np.asarray(arr, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError('expected a 2-D array')
        r, c = np.nonzero(arr)
        return cls.from_coo(arr.shape[0], arr.shape[1], r, c, arr[r, c])

    @classmethod
    def identity(cls, n):
        return cls.csr(n, n, np.arange(n + 1), np.arange(n), np.ones(n), check=False)

    @property
    def nnz(self):
        return int(self.col_indices.numel())

    def to_host(self):
        """(row_offsets int64, col_indices int64, values float64) numpy arrays."""
        return (self.row_offsets.cpu().numpy().astype(np.int64),
                self.col_indices.cpu().numpy().astype(np.int64),
                self.values.cpu().numpy())

    def to_dense(self):
        p, c, v = self.to_host()
        out = np.zeros((self.nrows, self.ncols))
        out[np.repeat(np.arange(self.nrows), np.diff(p)), c] = v
        return out

    def row(self, i):
        p, c, v = self.to_host()
        return c[p[i]:p[i + 1]], v[p[i]:p[i + 1]]

    def __repr__(self):
        return f'SparseMatrix({self.nrows}x{self.ncols}, nnz={self.nnz}, device)'


def validate(A):
    """Canonical-form invariants (sparse.py:183-203); raises ValueError."""
    p, c, v = A.to_host()
    if A.nrows < 0 or A.ncols < 0:
        raise ValueError('negative dimension')
    if len(p) != A.nrows + 1:
        raise ValueError('row_offsets has wrong length')
    if p[0] != 0 or p[-1] != len(c) or len(c) != len(v):
        raise ValueError('row_offsets endpoints inconsistent with entry arrays')
    if np.any(np.diff(p) < 0):
        raise ValueError('row_offsets must be non-decreasing')
    if len(c):
        if c.min() < 0 or c.max() >= A.ncols:
            raise ValueError('column index out of range')
        r = np.repeat(np.arange(A.nrows), np.diff(p))
        same = r[1:] == r[:-1]
        if not np.all(c[1:][same] > c[:-1][same]):
            raise ValueError('column indices must be strictly increasing within rows')
    if len(v) and not np.all(np.isfinite(v)):
        raise ValueError('stored values must be finite')
    return A


def as_vector(x, n=None):
    t = to_dev(x, VAL)
    if t.dim() != 1 or (n is not None and t.numel() != n):
        raise ValueError(f'vector of length {t.numel()} incompatible with length {n}')
    return t


def spmv(A, x, exact=False):
    """y = A x (sparse.py:206-212).  ``exact=True`` reproduces scipy's
    sequential non-FMA row sums bitwise; the default is the vector kernel."""
    x = to_dev(x, VAL)
    if x.dim() != 1 or x.numel() != A.ncols:
        raise ValueError(f'vector of length {x.numel()} incompatible with '
                         f'{A.nrows}x{A.ncols} matrix')
    y = empty(A.nrows, VAL)
    L.call('airg_spmv', A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
           L.ptr(x), L.ptr(y), 1 if exact else 0, L.stream_handle())
    return y


def norm2(x):
    out = np.zeros(1)
    L.call('airg_norm2', x.numel(), L.ptr(x), L.hptr(out), L.stream_handle())
    return float(out[0])
