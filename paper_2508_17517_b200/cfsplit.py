"""Strength graph, PMISR Luby independent set and DDC cleanup on the GPU
(ref: splitting.py:15-238).

Luby weights are numpy's PCG64 stream reproduced per element on the device
(jump-ahead), so the F/C labels are bit-identical to the reference's.
"""

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .csr import IDX, SparseMatrix, empty, take, to_dev

F_POINT = 0
C_POINT = 1


@dataclass(frozen=True, eq=False)
class CFSplit:
    """Per-unknown F/C labels with sorted index sets (splitting.py:46-71).

    ``labels`` (int8), ``f_idx`` / ``c_idx`` / ``pos`` (int32) are device
    tensors (``pos[i]`` = rank of i inside its class); ``f_set`` / ``c_set``
    give the reference's host int64 views.
    """

    labels: torch.Tensor
    f_idx: torch.Tensor
    c_idx: torch.Tensor
    pos: torch.Tensor

    @classmethod
    def from_labels(cls, labels):
        lab = to_dev(labels, torch.int8)
        n = lab.numel()
        nf = C.c_int32()
        pos = empty(n, IDX)
        L.call('airg_split_index', n, L.ptr(lab), L.ptr(pos), None, None, C.byref(nf),
               L.stream_handle())
        f = empty(nf.value, IDX)
        c = empty(n - nf.value, IDX)
        L.call('airg_split_index', n, L.ptr(lab), None, L.ptr(f), L.ptr(c), C.byref(nf),
               L.stream_handle())
        return cls(lab, f, c, pos)

    @property
    def n(self):
        return int(self.labels.numel())

    @property
    def n_f(self):
        return int(self.f_idx.numel())

    @property
    def n_c(self):
        return int(self.c_idx.numel())

    @property
    def f_set(self):
        return self.f_idx.cpu().numpy().astype(np.int64)

    @property
    def c_set(self):
        return self.c_idx.cpu().numpy().astype(np.int64)

    def labels_host(self):
        return self.labels.cpu().numpy()


@dataclass(frozen=True)
class StrengthGraph:
    """Strong connections S and the pattern of S + S^T (splitting.py:33-43)."""

    S: SparseMatrix
    symmetric_closure: SparseMatrix

    @property
    def n(self):
        return self.S.nrows


@dataclass(frozen=True)
class DDCPassStats:
    """Diagnostics from one diagonal-dominance cleanup pass (splitting.py:74-83)."""

    n_f_before: int
    converted: int
    ratio_min: float
    ratio_max: float
    ratio_mean: float
    cut: float


def _square(A, what):
    if A.nrows != A.ncols:
        raise ValueError(f'{what} requires a square matrix')


def strength_graph(A, theta):
    """Edge (i, j) iff j != i, a_ij != 0, |a_ij| >= theta max_{k!=i} |a_ik|
    (splitting.py:86-109)."""
    _square(A, 'strength graph')
    if not 0.0 <= theta <= 1.0:
        raise ValueError('theta must lie in [0, 1]')
    s, c = C.c_void_p(), C.c_void_p()
    L.call('airg_strength', A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
           A.nnz, float(theta), C.byref(s), C.byref(c), L.stream_handle())
    return StrengthGraph(take(s), take(c))


def pmisr(graph, seed, max_luby_loops=None):
    """Luby rounds on the symmetric closure; independent set -> F (splitting.py:127-159)."""
    G = graph.symmetric_closure
    labels = empty(G.nrows, torch.int8)
    loops = C.c_int32()
    L.call('airg_pmisr', G.nrows, L.ptr(G.row_offsets), L.ptr(G.col_indices),
           *L.pcg_params(seed), -1 if max_luby_loops is None else int(max_luby_loops),
           L.ptr(labels), C.byref(loops), L.stream_handle())
    return CFSplit.from_labels(labels)


def _cf_labels(A, theta, seed, max_luby_loops=None):
    """strength + closure + PMISR in one library call; returns device labels."""
    labels = empty(A.nrows, torch.int8)
    loops = C.c_int32()
    L.call('airg_cf_pmisr', A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices),
           L.ptr(A.values), A.nnz, float(theta), *L.pcg_params(seed),
           -1 if max_luby_loops is None else int(max_luby_loops), L.ptr(labels), C.byref(loops),
           L.stream_handle())
    return labels


def _ddc_labels(A, labels, fraction, nbins):
    """One DDC pass on device labels (in place); returns DDCPassStats."""
    st = np.zeros(6)
    L.call('airg_ddc_pass', A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
           L.ptr(labels), float(fraction), int(nbins), L.hptr(st), L.stream_handle())
    return DDCPassStats(n_f_before=int(st[0]), converted=int(st[1]), ratio_min=float(st[2]),
                        ratio_max=float(st[3]), ratio_mean=float(st[4]), cut=float(st[5]))


def _ddc_core(A, split, fraction, nbins):
    if not 0.0 < fraction < 1.0:
        raise ValueError('fraction must lie in (0, 1)')
    if nbins < 1:
        raise ValueError('nbins must be positive')
    _square(A, 'diagonal-dominance cleanup')
    lab = split.labels.clone()
    stats = _ddc_labels(A, lab, fraction, nbins)
    return CFSplit.from_labels(lab), stats


def ddc_pass(A, split, fraction, nbins=1000):
    """One diagonal-dominance cleanup pass (splitting.py:210-216)."""
    return _ddc_core(A, split, fraction, nbins)[0]


def cf_split(A, theta, ddc_fraction, ddc_its, seed, nbins=1000, max_luby_loops=None):
    """Strength -> PMISR -> ddc_its DDC passes (splitting.py:219-238).

    Returns (CFSplit, [DDCPassStats])."""
    _square(A, 'strength graph')
    if not 0.0 <= theta <= 1.0:
        raise ValueError('theta must lie in [0, 1]')
    labels = _cf_labels(A, theta, seed, max_luby_loops)
    stats = []
    nf = None
    for _ in range(ddc_its):
        if nf is None:
            nf = int((labels == F_POINT).sum().item())
        if nf == 0:
            break
        if not 0.0 < ddc_fraction < 1.0:
            raise ValueError('fraction must lie in (0, 1)')
        st = _ddc_labels(A, labels, ddc_fraction, nbins)
        stats.append(st)
        nf = st.n_f_before - st.converted
    return CFSplit.from_labels(labels), stats
