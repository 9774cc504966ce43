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


def dg_q1_blocks(hx, hy, vx, vy):
    """4x4 cell blocks of the upwind DG operator for v . grad u on a uniform
    hx x hy cell with the nodal Q1 basis psi_k = l_s(xi) l_t(eta), k = s + 2t,
    l_0 = (1 - t)/2, l_1 = (1 + t)/2 (Lagrange at the cell corners) -- the
    basis AIR is normally applied with (a modal Legendre basis was measured
    to need 34 vs 12 iterations at 128^2 cells and to diverge at 512^2).
    Row = test node a, column = trial node b.  Weak form per cell:
    -int u v.grad(psi) + outflow-face int (v.n) u psi + inflow-face
    int (v.n) u_upwind psi, in closed form (int l_i l_j = 2/3 or 1/3,
    int l_j l_i' = -+1/2, traces l_i(+-1) in {0, 1}): D = own cell (volume +
    east/north outflow faces), W / S = west / south neighbour (inflow faces;
    only the nodes on the shared face couple)."""
    import numpy as np
    M = ((2.0 / 3.0, 1.0 / 3.0), (1.0 / 3.0, 2.0 / 3.0))
    dl = (-0.5, 0.5)  # int l_j l_i' (independent of j)
    ax, ay = vx * hy / 2.0, vy * hx / 2.0
    D, W, S = np.zeros((4, 4)), np.zeros((4, 4)), np.zeros((4, 4))
    for a in range(4):
        sa, ta = a % 2, a // 2
        for b in range(4):
            sb, tb = b % 2, b // 2
            vol = -(ax * dl[sa] * M[tb][ta]) - ay * M[sb][sa] * dl[ta]
            east = ax * M[tb][ta] if (sa == 1 and sb == 1) else 0.0
            north = ay * M[sb][sa] if (ta == 1 and tb == 1) else 0.0
            D[a, b] = vol + east + north
            W[a, b] = -ax * M[tb][ta] if (sa == 0 and sb == 1) else 0.0
            S[a, b] = -ay * M[sb][sa] if (ta == 0 and tb == 1) else 0.0
    return D, W, S


def build_advection_dg(problem):
    """Upwind DG (nodal Q1, 4 unknowns per cell) operator of the problem's velocity
    on its nx x ny cells and the zero right-hand side (homogeneous inflow
    data), generated in HBM.  SURVEY 8(d) cfg 5: the reference has no DG
    generator; the problem class and velocity convention are its
    (problems.py:20-45)."""
    import numpy as np
    from .csr import take
    p = problem
    if p.ny < 1:
        raise ValueError('build_advection_dg requires ny >= 1')
    D, W, S = dg_q1_blocks(p.Lx / p.nx, p.Ly / p.ny, float(p.vx), float(p.vy))
    blk = np.ascontiguousarray(np.concatenate([D.ravel(), W.ravel(), S.ravel()]))
    res = L.C.c_void_p()
    L.call('airg_advection_dg', p.nx, p.ny, L.hptr(blk), int(p.vx > 0), int(p.vy > 0),
           L.C.byref(res), L.stream_handle())
    A = take(res)
    return A, torch.zeros(A.nrows, dtype=VAL, device=A.values.device)
