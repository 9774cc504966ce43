"""Device CSR container and the sparse kernels of the AIRG path.

Mirrors the reference's ``airmg.sparse`` interface (sparse.py:18-30, 44-367):
``SparseMatrix``, ``validate``, ``spmv``, ``spgemm``, ``spgemm_fixed_sparsity``,
``extract``, ``drop_and_lump``, ``diagonal``.  Storage lives in HBM as
int32 row offsets / int32 columns / fp64 values (torch tensors used only as
device buffers); every operation is an sm_100a kernel in libairg.so.
"""

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

IDX = torch.int32
VAL = torch.float64


_HAVE_CUDA = False


def _dev():
    global _HAVE_CUDA
    if not _HAVE_CUDA:  # checked until a device is seen (then once per process)
        if not torch.cuda.is_available():
            raise RuntimeError('paper_2508_17517_b200 needs a CUDA device (sm_100a); '
                               'there is no CPU fallback')
        _HAVE_CUDA = True
    return torch.device('cuda', torch._C._cuda_getDevice())


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


def as_matrix(A):
    """The device form of ``A``: a SparseMatrix passes through; a host CSR
    object with the reference's attributes (``airmg.SparseMatrix``:
    nrows, ncols, int64 row_offsets / col_indices, float64 values --
    sparse.py:44-73) is uploaded, so reference callers can pass their own
    matrices.  Indices must fit int32 (the device CSR's index type)."""
    if isinstance(A, SparseMatrix):
        return A
    try:
        nr, nc = int(A.nrows), int(A.ncols)
        p, c, v = A.row_offsets, A.col_indices, A.values
    except AttributeError:
        raise TypeError(f'expected a CSR matrix (nrows, ncols, row_offsets, col_indices, values), '
                        f'got {type(A).__name__}') from None
    p = np.asarray(p) if not isinstance(p, torch.Tensor) else p
    if max(nr, nc, int(p[-1]) if len(p) else 0) > np.iinfo(np.int32).max:
        raise ValueError('matrix too large for 32-bit device indices')
    return SparseMatrix.csr(nr, nc, p, c, v, check=False)


def is_host_array(x):
    """True for inputs the reference API takes as numpy arrays (not device tensors)."""
    return not isinstance(x, torch.Tensor)


def as_vector(x, n=None):
    t = to_dev(x, VAL)
    if t.dim() != 1 or (n is not None and t.numel() != n):
        raise ValueError(f'vector of length {t.numel()} incompatible with length {n}')
    return t


def spmv(A, x, exact=False):
    """y = A x (sparse.py:206-212).  ``exact=True`` reproduces scipy's
    sequential non-FMA row sums bitwise; the default is the vector kernel."""
    A = as_matrix(A)
    x = to_dev(x, VAL)
    if x.dim() != 1 or x.numel() != A.ncols:
        raise ValueError(f'vector of length {x.numel()} incompatible with '
                         f'{A.nrows}x{A.ncols} matrix')
    y = empty(A.nrows, VAL)
    L.call('airg_spmv', A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
           L.ptr(x), L.ptr(y), 1 if exact else 0, L.stream_handle())
    return y


@dataclass(frozen=True, eq=False)
class EllMatrix:
    """Fixed-width (ELL) copy of a CSR matrix for the structured stencils:
    ``cols`` / ``vals`` hold ``width`` slots per row, column-major."""

    nrows: int
    ncols: int
    width: int
    cols: torch.Tensor
    vals: torch.Tensor


def to_ell(A, width=None):
    """CSR -> ELL (width = longest row unless given)."""
    lens = A.row_offsets[1:] - A.row_offsets[:-1]
    w = int(lens.max().item()) if width is None and A.nrows else int(width or 0)
    cols = empty(max(A.nrows * w, 1), IDX)
    vals = empty(max(A.nrows * w, 1), VAL)
    L.call('airg_csr_to_ell', A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
           w, L.ptr(cols), L.ptr(vals), L.stream_handle())
    return EllMatrix(A.nrows, A.ncols, w, cols, vals)


def spmv_ell(E, x, exact=False):
    """y = A x on the ELL copy; ``exact=True`` is bitwise ``spmv(A, x, exact=True)``."""
    x = to_dev(x, VAL)
    if x.dim() != 1 or x.numel() != E.ncols:
        raise ValueError(f'vector of length {x.numel()} incompatible with '
                         f'{E.nrows}x{E.ncols} matrix')
    y = empty(E.nrows, VAL)
    L.call('airg_spmv_ell', E.nrows, E.width, L.ptr(E.cols), L.ptr(E.vals), L.ptr(x), L.ptr(y),
           1 if exact else 0, L.stream_handle())
    return y


def norm2(x):
    out = np.zeros(1)
    L.call('airg_norm2', x.numel(), L.ptr(x), L.hptr(out), L.stream_handle())
    return float(out[0])


# ---------------------------------------------------------------------------
# variable-size results
# ---------------------------------------------------------------------------

def new_result():
    return C.c_void_p()


class _LibBuffer:
    """A library-pool device buffer seen by torch without a copy
    (__cuda_array_interface__; torch keeps this object alive as long as the
    tensor).  Returned to the pool, on the then-current stream, when the last
    tensor viewing it dies."""

    __slots__ = ('ptr', 'n', 'typestr', '__weakref__')

    def __init__(self, ptr, n, typestr):
        self.ptr, self.n, self.typestr = ptr, n, typestr

    @property
    def __cuda_array_interface__(self):
        return {'shape': (self.n,), 'typestr': self.typestr, 'data': (self.ptr, False),
                'version': 3, 'strides': None}

    def __del__(self):
        try:
            L.load().airg_buffer_free(C.c_void_p(self.ptr), L.stream_handle())
        except Exception:  # interpreter shutdown
            pass


def _view(ptr, n, dtype):
    typestr = {IDX: '<i4', VAL: '<f8'}[dtype]
    return torch.as_tensor(_LibBuffer(ptr, n, typestr), device=_dev())


_TAKE_COPY = bool(os.environ.get('AIRG_TAKE_COPY'))


def take(res, values=True):
    """Adopt a library-held airg_csr_result as device tensors (zero-copy:
    the result's pool buffers become the tensors' storage; AIRG_TAKE_COPY=1
    copies into torch-allocated tensors instead)."""
    nr, nc, nnz = C.c_int32(), C.c_int32(), C.c_int64()
    L.call('airg_result_info', res, C.byref(nr), C.byref(nc), C.byref(nnz))
    if _TAKE_COPY:
        p = empty(nr.value + 1, IDX)
        c = empty(nnz.value, IDX)
        v = empty(nnz.value, VAL) if values else None
        L.call('airg_result_take', res, L.ptr(p), L.ptr(c), L.ptr(v), L.stream_handle())
        if v is None:
            v = torch.ones(nnz.value, dtype=VAL, device=p.device)
        return SparseMatrix(nr.value, nc.value, p, c, v)
    pp, pc, pv = C.c_void_p(), C.c_void_p(), C.c_void_p()
    L.call('airg_result_detach', res, C.byref(pp), C.byref(pc), C.byref(pv), L.stream_handle())
    p = _view(pp.value, nr.value + 1, IDX)
    c = _view(pc.value, nnz.value, IDX) if pc.value else empty(nnz.value, IDX)
    if values and pv.value:
        v = _view(pv.value, nnz.value, VAL)
    else:
        if pv.value:
            L.load().airg_buffer_free(pv, L.stream_handle())
        v = (torch.zeros if values else torch.ones)(nnz.value, dtype=VAL, device=p.device)
    return SparseMatrix(nr.value, nc.value, p, c, v)


def _args(A):
    return L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values)


def spgemm(A, B, negate=False):
    """Structural product, cancellation zeros kept (sparse.py:222-240)."""
    A, B = as_matrix(A), as_matrix(B)
    if A.ncols != B.nrows:
        raise ValueError(f'cannot multiply {A.nrows}x{A.ncols} by {B.nrows}x{B.ncols}')
    r = new_result()
    L.call('airg_spgemm', A.nrows, A.ncols, B.ncols, *_args(A), *_args(B), 1 if negate else 0,
           C.byref(r), L.stream_handle())
    return take(r)


def spgemm_fixed_sparsity(A, B, pattern):
    """A @ B restricted to the stored positions of ``pattern`` (sparse.py:243-263)."""
    A, B, pattern = as_matrix(A), as_matrix(B), as_matrix(pattern)
    if A.ncols != B.nrows:
        raise ValueError(f'cannot multiply {A.nrows}x{A.ncols} by {B.nrows}x{B.ncols}')
    if pattern.nrows != A.nrows or pattern.ncols != B.ncols:
        raise ValueError('pattern shape must match the product shape')
    r = new_result()
    L.call('airg_spgemm_masked', A.nrows, A.ncols, B.ncols, *_args(A), *_args(B),
           L.ptr(pattern.row_offsets), L.ptr(pattern.col_indices), C.byref(r), L.stream_handle())
    return take(r)


def _index_set(idx, limit, name):
    t = to_dev(idx, IDX)
    if t.dim() != 1:
        raise ValueError(f'{name} index set must be one-dimensional')
    if t.numel():
        h = t.cpu().numpy()
        if h[0] < 0 or h[-1] >= limit:
            raise ValueError(f'{name} index out of range for dimension {limit}')
        if np.any(np.diff(h) <= 0):
            raise ValueError(f'{name} index set must be strictly increasing')
    return t


def extract_mapped(A, rows, colmap, ncols):
    """A[rows, :] with columns renumbered through ``colmap`` (-1 drops)."""
    r = new_result()
    L.call('airg_extract_ex', int(rows.numel()), L.ptr(rows), *_args(A), L.ptr(colmap), int(ncols),
           A.nnz / max(A.nrows, 1), C.byref(r), L.stream_handle())
    return take(r)


def extract(A, rows, cols):
    """Submatrix A[rows, cols], renumbered, entry order kept (sparse.py:278-304)."""
    A = as_matrix(A)
    rows = _index_set(rows, A.nrows, 'row')
    cols = _index_set(cols, A.ncols, 'column')
    colmap = torch.full((A.ncols,), -1, dtype=IDX, device=rows.device)
    colmap[cols.long()] = torch.arange(cols.numel(), dtype=IDX, device=rows.device)
    return extract_mapped(A, rows, colmap, cols.numel())


def drop_and_lump(A, rel_tol, lump):
    """Row-relative drop, optional sequential lump onto the diagonal (sparse.py:307-352)."""
    A = as_matrix(A)
    if rel_tol < 0:
        raise ValueError('rel_tol must be non-negative')
    if lump and A.nrows != A.ncols:
        raise ValueError('lumping requires a square matrix')
    if rel_tol == 0 or A.nnz == 0:
        return A
    r = new_result()
    changed = C.c_int32()
    L.call('airg_drop_lump', A.nrows, A.ncols, *_args(A), float(rel_tol), 1 if lump else 0,
           C.byref(r), C.byref(changed), L.stream_handle())
    out = take(r)
    return out if changed.value else A


def diagonal(A):
    """Main diagonal as a device vector (sparse.py:360-367)."""
    A = as_matrix(A)
    n = min(A.nrows, A.ncols)
    d = empty(n, VAL)
    L.call('airg_diagonal', n, *_args(A), L.ptr(d), L.stream_handle())
    return d


def pcg_vector(seed, n, a, b):
    """out[i] = a + b * Generator(PCG64(SeedSequence(seed))).random()_i, on the GPU."""
    out = empty(n, VAL)
    L.call('airg_pcg64_fill', *L.pcg_params(seed), int(n), float(a), float(b), L.ptr(out),
           L.stream_handle())
    return out


def random_unit_vector(n, seed):
    """uniform(-1, 1, n) normalised (polynomial.py:61-65), generated on the GPU."""
    out = empty(n, VAL)
    L.call('airg_random_unit', *L.pcg_params(seed), int(n), L.ptr(out), None, L.stream_handle())
    return out


def write_matrix_market(A, path):
    """Matrix Market coordinate real general, values with 17 significant
    digits (exact float64 round trip).  ref: sparse.py:370-381"""
    p, c, v = A.to_host()
    rows = np.repeat(np.arange(A.nrows), np.diff(p)) + 1
    with open(path, 'w') as fh:
        fh.write('%%MatrixMarket matrix coordinate real general\n')
        fh.write(f'{A.nrows} {A.ncols} {len(v)}\n')
        fh.writelines(f'{i} {j} {x:.16e}\n' for i, j, x in zip(rows, c + 1, v))


def read_matrix_market(path):
    """Read a Matrix Market coordinate real general file into a device CSR
    (duplicates summed, sorted columns).  ref: sparse.py:384-410"""
    with open(path) as fh:
        banner = fh.readline().split()
        if (len(banner) != 5 or banner[0] != '%%MatrixMarket'
                or [t.lower() for t in banner[1:]] != ['matrix', 'coordinate', 'real', 'general']):
            raise ValueError('expected a "matrix coordinate real general" file')
        line = fh.readline()
        while line.startswith('%'):
            line = fh.readline()
        dims = line.split()
        if len(dims) != 3:
            raise ValueError('malformed size line')
        nrows, ncols, nnz = (int(t) for t in dims)
        body = np.loadtxt(fh, comments='%', ndmin=2) if nnz else np.zeros((0, 3))
    if body.size == 0:
        body = body.reshape(0, 3)
    if body.shape[0] != nnz or (nnz and body.shape[1] != 3):
        raise ValueError('entry count does not match the size line')
    return SparseMatrix.from_coo(nrows, ncols, body[:, 0].astype(np.int64) - 1,
                                 body[:, 1].astype(np.int64) - 1, body[:, 2])
