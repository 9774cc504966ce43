"""Strength graph, PMISR Luby independent set and DDC cleanup on the GPU
(ref: splitting.py:15-238)."""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .csr import IDX, SparseMatrix, empty, to_dev

F_POINT = 0
C_POINT = 1


@dataclass(frozen=True, eq=False)
class CFSplit:
    """Per-unknown F/C labels with sorted index sets (splitting.py:46-71).

    ``labels`` (int8), ``f_idx`` / ``c_idx`` (int32) are device tensors;
    ``f_set`` / ``c_set`` give the reference's host int64 views.
    """

    labels: torch.Tensor
    f_idx: torch.Tensor
    c_idx: torch.Tensor

    @classmethod
    def from_labels(cls, labels):
        lab = to_dev(labels, torch.int8)
        f = torch.nonzero(lab == F_POINT).flatten().to(IDX)
        c = torch.nonzero(lab == C_POINT).flatten().to(IDX)
        return cls(lab, f, c)

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
