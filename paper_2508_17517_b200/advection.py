"""Upwind advection test operators generated directly in HBM
(ref: problems.py:17-99).  Unknown (i, j) is index j*nx + i; rows hold
south (-vy), west (-vx), diagonal (vx + vy) in column order."""

from dataclasses import dataclass

import torch

from . import _lib as L
from .csr import IDX, VAL, SparseMatrix, empty


@dataclass(frozen=True)
class AdvectionProblem:
    """Constant-velocity advection on an nx x ny grid (problems.py:20-45)."""

    nx: int
    ny: int
    vx: float
    vy: float
    Lx: float = 1.0
    Ly: float = 1.0

    def __post_init__(self):
        if self.nx < 1 or self.ny < 0:
            raise ValueError('require nx >= 1 and ny >= 0')
        if self.vx < 0 or self.vy < 0 or self.vx + self.vy <= 0:
            raise ValueError('velocity must satisfy vx >= 0, vy >= 0, vx + vy > 0')

    @property
    def n(self):
        return self.nx * max(self.ny, 1)


def _generate(nx, ny, vx, vy):
    n = nx * ny
    nnz = n + (nx - 1) * ny * (vx > 0) + nx * (ny - 1) * (vy > 0)
    p, c, v = empty(n + 1, IDX), empty(nnz, IDX), empty(nnz, VAL)
    L.call('airg_advection_2d', nx, ny, float(vx), float(vy), L.ptr(p), L.ptr(c), L.ptr(v),
           L.stream_handle())
    return SparseMatrix(n, n, p, c, v)


def build_advection_2d(problem):
    """2-D upwind operator and its zero right-hand side (problems.py:48-85)."""
    p = problem
    if p.ny < 1:
        raise ValueError('build_advection_2d requires ny >= 1; use build_advection_1d for 1-D '
                         'problems')
    A = _generate(p.nx, p.ny, float(p.vx), float(p.vy))
    return A, torch.zeros(A.nrows, dtype=VAL, device=A.values.device)


def build_advection_1d(n, vx):
    """Lower bidiagonal 1-D upwind operator (problems.py:88-99)."""
    if n < 1:
        raise ValueError('require n >= 1')
    if vx <= 0:
        raise ValueError('require vx > 0')
    return _generate(int(n), 1, float(vx), 0.0)
