"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the AIRG setup + solve path.

This module is the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product (``paper_2508_17517_b200``) never does; it runs sm_100a kernels.

It restates, in numpy/scipy, the algorithm of the reference package ``airmg``
(``/root/reference/pkg/src/airmg``; cited below as ``sparse.py:N`` etc.).  The
arithmetic that defines bit-level results lives in third-party code the
reference calls, and the oracle calls the same routines in the same order:

* scipy 1.18 sparsetools ``csr_matvec`` / ``csr_matmat`` (sequential,
  k-ascending, no FMA) and ``csr_binop_csr`` (prunes exact zeros);
* numpy 2.3 ``PCG64``/``SeedSequence`` streams, ``bincount`` (sequential);
* OpenBLAS ddot/dnrm2 and LAPACK gelsd/gesdd/gesv/geev for the small dense
  Krylov algebra (thread-count dependent rounding -- pin
  ``OPENBLAS_NUM_THREADS=1`` when comparing with a fixture).

Pinning: ``tests/golden/make_golden.py`` imports the reference in this
container and writes fixtures; ``tests/test_oracle_golden.py`` proves the
oracle reproduces them bit for bit.

Extra hooks the reference does not have (test-only):

* ``setup(..., poly_inject=...)`` -- coefficient injection: the smoother /
  coarse polynomials are taken from a dict instead of being recomputed, so a
  hierarchy built on the GPU (whose Krylov dot products round differently)
  can be replayed exactly here.
* ``setup(..., keep_level_matrices=True)`` keeps every level matrix A_l.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sps

I64 = np.int64
F64 = np.float64

# --------------------------------------------------------------------------
# CSR container (sparse.py:44-152)
# --------------------------------------------------------------------------


@dataclass(frozen=True, eq=False)
class Csr:
    nrows: int
    ncols: int
    ptr: np.ndarray   # int64[nrows+1]
    col: np.ndarray   # int64[nnz], strictly increasing per row
    val: np.ndarray   # float64[nnz]

    @property
    def nnz(self):
        return int(self.ptr[-1])

    def sp(self):
        m = sps.csr_matrix((self.val, self.col, self.ptr),
                           shape=(self.nrows, self.ncols), copy=False)
        m.has_sorted_indices = True
        return m

    def rows(self):
        return np.repeat(np.arange(self.nrows, dtype=I64), np.diff(self.ptr))

    def dense(self):
        out = np.zeros((self.nrows, self.ncols))
        out[self.rows(), self.col] = self.val
        return out


def _mk(nrows, ncols, ptr, col, val):
    return Csr(int(nrows), int(ncols), np.ascontiguousarray(ptr, dtype=I64),
               np.ascontiguousarray(col, dtype=I64),
               np.ascontiguousarray(val, dtype=F64))


def ptr_from_rows(row_ids, nrows):
    ptr = np.zeros(nrows + 1, dtype=I64)
    np.cumsum(np.bincount(row_ids, minlength=nrows), out=ptr[1:])
    return ptr


def from_triplets(nrows, ncols, r, c, v):
    """COO -> canonical CSR, duplicates summed in sorted order (sparse.py:75-97)."""
    r = np.asarray(r, dtype=I64)
    c = np.asarray(c, dtype=I64)
    v = np.asarray(v, dtype=F64)
    o = np.lexsort((c, r))
    r, c, v = r[o], c[o], v[o]
    if len(r):
        head = np.ones(len(r), dtype=bool)
        head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        s = np.flatnonzero(head)
        v = np.add.reduceat(v, s)
        r, c = r[s], c[s]
    return _mk(nrows, ncols, ptr_from_rows(r, nrows), c, v)


def from_scipy(m):
    """Wrap a scipy CSR result, sorting rows that came back unsorted (sparse.py:107-118)."""
    m = m.tocsr()
    ptr = np.asarray(m.indptr, dtype=I64)
    col = np.asarray(m.indices, dtype=I64)
    val = np.asarray(m.data, dtype=F64)
    nr = m.shape[0]
    rows = np.repeat(np.arange(nr, dtype=I64), np.diff(ptr))
    if len(col) > 1:
        same = rows[1:] == rows[:-1]
        if not np.all(col[1:][same] > col[:-1][same]):
            o = np.lexsort((col, rows))
            col, val = col[o], val[o]
    return _mk(nr, m.shape[1], ptr, col, val)


def identity(n):
    return _mk(n, n, np.arange(n + 1), np.arange(n), np.ones(n))


def row_max(vals, ptr, nrows, empty=0.0):
    """Per-row max over stored entries (sparse.py:158-171)."""
    out = np.full(nrows, empty, dtype=F64)
    nz = np.diff(ptr) > 0
    if nz.any():
        out[nz] = np.maximum.reduceat(vals, ptr[:-1][nz])
    return out


def keys(A):
    return A.rows() * I64(A.ncols) + A.col if A.nnz else np.zeros(0, dtype=I64)


# --------------------------------------------------------------------------
# kernels (sparse.py:206-367)
# --------------------------------------------------------------------------


def spmv(A, x):
    return A.sp() @ np.asarray(x, dtype=F64)


def spgemm(A, B):
    """Structural product; cancellation zeros kept as +0.0 (sparse.py:222-240)."""
    ones_a = sps.csr_matrix((np.ones(A.nnz), A.col, A.ptr), shape=(A.nrows, A.ncols))
    ones_b = sps.csr_matrix((np.ones(B.nnz), B.col, B.ptr), shape=(B.nrows, B.ncols))
    pat = from_scipy(ones_a @ ones_b)
    num = from_scipy(A.sp() @ B.sp())
    if num.nnz == pat.nnz:
        return num
    v = np.zeros(pat.nnz)
    v[np.searchsorted(keys(pat), keys(num))] = num.val
    return _mk(pat.nrows, pat.ncols, pat.ptr, pat.col, v)


def spgemm_masked(A, B, P):
    """A@B kept only at stored positions of P (sparse.py:243-263)."""
    prod = spgemm(A, B)
    pk, qk = keys(P), keys(prod)
    pos = np.searchsorted(pk, qk)
    ok = pos < len(pk)
    keep = np.zeros(prod.nnz, dtype=bool)
    keep[ok] = pk[pos[ok]] == qk[ok]
    return _mk(prod.nrows, prod.ncols, ptr_from_rows(prod.rows()[keep], prod.nrows),
               prod.col[keep], prod.val[keep])


def submatrix(A, rows, cols):
    """A[rows, cols] renumbered, entry order preserved (sparse.py:278-304)."""
    rows = np.asarray(rows, dtype=I64)
    cols = np.asarray(cols, dtype=I64)
    member = np.full(A.ncols, -1, dtype=I64)
    member[cols] = np.arange(len(cols), dtype=I64)
    starts = A.ptr[rows]
    lens = A.ptr[rows + 1] - starts
    first = np.cumsum(lens) - lens
    take = (np.arange(int(lens.sum()), dtype=I64) - np.repeat(first, lens)
            + np.repeat(starts, lens))
    newcol = member[A.col[take]]
    keep = newcol >= 0
    rid = np.repeat(np.arange(len(rows), dtype=I64), lens)[keep]
    return _mk(len(rows), len(cols), ptr_from_rows(rid, len(rows)), newcol[keep],
               A.val[take][keep])


def diag_of(A):
    n = min(A.nrows, A.ncols)
    out = np.zeros(n)
    r = A.rows()
    hit = (A.col == r) & (r < n)
    out[r[hit]] = A.val[hit]
    return out


def drop_lump(A, tol, lump):
    """Row-relative drop, sequential lump onto the diagonal (sparse.py:307-352)."""
    if tol < 0:
        raise ValueError('rel_tol must be non-negative')
    if lump and A.nrows != A.ncols:
        raise ValueError('lumping requires a square matrix')
    if tol == 0 or A.nnz == 0:
        return A
    r = A.rows()
    mag = np.abs(A.val)
    rmax = row_max(mag, A.ptr, A.nrows)
    ondiag = A.col == r
    keep = ondiag | (mag >= tol * rmax[r])
    if keep.all():
        return A
    if not lump:
        return _mk(A.nrows, A.ncols, ptr_from_rows(r[keep], A.nrows), A.col[keep], A.val[keep])
    lumped = np.bincount(r[~keep], weights=A.val[~keep], minlength=A.nrows)
    kr, kc, kv = r[keep], A.col[keep], A.val[keep].copy()
    dpos = kc == kr
    kv[dpos] += lumped[kr[dpos]]
    has = np.zeros(A.nrows, dtype=bool)
    has[kr[dpos]] = True
    ins = np.flatnonzero(~has & (lumped != 0))
    if len(ins):
        return from_triplets(A.nrows, A.ncols, np.concatenate([kr, ins]),
                             np.concatenate([kc, ins]), np.concatenate([kv, lumped[ins]]))
    return _mk(A.nrows, A.ncols, ptr_from_rows(kr, A.nrows), kc, kv)


# --------------------------------------------------------------------------
# problems (problems.py:48-99)
# --------------------------------------------------------------------------


def advection_2d(nx, ny, vx, vy):
    n = nx * ny
    idx = np.arange(n, dtype=I64)
    i, j = idx % nx, idx // nx
    rs, cs, vs = [idx], [idx], [np.full(n, vx + vy)]
    if vx > 0:
        w = idx[i > 0]
        rs.append(w); cs.append(w - 1); vs.append(np.full(len(w), -vx))
    if vy > 0:
        s = idx[j > 0]
        rs.append(s); cs.append(s - nx); vs.append(np.full(len(s), -vy))
    return from_triplets(n, n, np.concatenate(rs), np.concatenate(cs), np.concatenate(vs))


def advection_dg_q1(nx, ny, vx, vy, Lx=1.0, Ly=1.0):
    """Upwind DG operator, nodal Q1 (SURVEY 8(d) cfg 5 -- no reference
    generator, so this is the specification): per cell e = j*nx + i, unknowns
    4e + k at the corners, psi_k = l_s(xi) l_t(eta), k = s + 2t, l_0 =
    (1 - t)/2, l_1 = (1 + t)/2.  Row (e, a): -int psi_b v.grad(psi_a) +
    east/north outflow-face terms on the own cell; west/south inflow-face
    terms on the upwind neighbour's face nodes (their traces at xi = 1 /
    eta = 1); exact zeros not stored."""
    hx, hy = Lx / nx, Ly / ny
    M = ((2.0 / 3.0, 1.0 / 3.0), (1.0 / 3.0, 2.0 / 3.0))   # int l_i l_j
    dl = (-0.5, 0.5)                                       # int l_j l_i'
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
    n = 4 * nx * ny
    rs, cs, vs = [], [], []
    e = np.arange(nx * ny, dtype=I64)
    i, j = e % nx, e // nx
    for blk, ok, nbr in ((S, (j > 0) & (vy > 0), e - nx), (W, (i > 0) & (vx > 0), e - 1),
                         (D, np.ones(nx * ny, dtype=bool), e)):
        for a in range(4):
            for b in range(4):
                if blk[a, b] != 0.0:
                    rs.append(4 * e[ok] + a)
                    cs.append(4 * nbr[ok] + b)
                    vs.append(np.full(int(ok.sum()), blk[a, b]))
    return from_triplets(n, n, np.concatenate(rs), np.concatenate(cs), np.concatenate(vs))


def dg_q1_blocks_gauss(hx, hy, vx, vy):
    """The same cell blocks by 2-point Gauss quadrature (exact for these
    degrees): an independent check of the closed forms above."""
    g = np.array([-1.0, 1.0]) / np.sqrt(3.0)
    l = (lambda t: (1 - t) / 2, lambda t: (1 + t) / 2)
    dlf = (lambda t: -0.5 * np.ones_like(t), lambda t: 0.5 * np.ones_like(t))
    X, Y = np.meshgrid(g, g, indexing='ij')
    one = np.array([1.0, 1.0])
    D, W, S = np.zeros((4, 4)), np.zeros((4, 4)), np.zeros((4, 4))
    for a in range(4):
        sa, ta = a % 2, a // 2
        for b in range(4):
            sb, tb = b % 2, b // 2
            psib = l[sb](X) * l[tb](Y)
            vol = -np.sum(psib * (vx * hy / 2 * dlf[sa](X) * l[ta](Y)
                                  + vy * hx / 2 * l[sa](X) * dlf[ta](Y)))
            east = vx * hy / 2 * np.sum(l[sb](one) * l[tb](g) * l[sa](one) * l[ta](g))
            north = vy * hx / 2 * np.sum(l[sb](g) * l[tb](one) * l[sa](g) * l[ta](one))
            D[a, b] = vol + east + north
            W[a, b] = -vx * hy / 2 * np.sum(l[sb](one) * l[tb](g) * l[sa](-one) * l[ta](g))
            S[a, b] = -vy * hx / 2 * np.sum(l[sb](g) * l[tb](one) * l[sa](g) * l[ta](-one))
    return D, W, S


def advection_1d(n, vx):
    idx = np.arange(n, dtype=I64)
    return from_triplets(n, n, np.concatenate([idx, idx[1:]]), np.concatenate([idx, idx[1:] - 1]),
                         np.concatenate([np.full(n, float(vx)), np.full(n - 1, -float(vx))]))


# --------------------------------------------------------------------------
# random streams (numpy PCG64; splitting.py:119, polynomial.py:63, hierarchy.py:52)
# --------------------------------------------------------------------------

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
M128 = (1 << 128) - 1
M64 = (1 << 64) - 1


def derive_seed(root, level, role):
    return int(np.random.SeedSequence([root, level, role]).generate_state(1)[0])


def pcg64_params(seed):
    st = np.random.PCG64(np.random.SeedSequence(seed)).state['state']
    return int(st['state']), int(st['inc'])


def pcg64_double_at(seed_state, inc, i):
    """Element i of Generator.random() by O(log i) LCG jump-ahead."""
    k = i + 1
    acc_m, acc_a, cm, ca = 1, 0, PCG_MULT, inc
    while k:
        if k & 1:
            acc_m = (acc_m * cm) & M128
            acc_a = (acc_a * cm + ca) & M128
        ca = ((cm + 1) * ca) & M128
        cm = (cm * cm) & M128
        k >>= 1
    s = (acc_m * seed_state + acc_a) & M128
    x = ((s >> 64) ^ s) & M64
    rot = s >> 122
    out = ((x >> rot) | (x << ((64 - rot) & 63))) & M64
    return (out >> 11) * (1.0 / 9007199254740992.0)


def uniform_unit(n, seed):
    v = np.random.default_rng(np.random.SeedSequence(seed)).uniform(-1.0, 1.0, n)
    return v / np.linalg.norm(v)


# --------------------------------------------------------------------------
# CF splitting (splitting.py:86-238)
# --------------------------------------------------------------------------

F_POINT, C_POINT = 0, 1


def strength(A, theta):
    n = A.nrows
    r = A.rows()
    off = A.col != r
    rmax = row_max(np.where(off, np.abs(A.val), 0.0), A.ptr, n)
    keep = off & (A.val != 0) & (np.abs(A.val) >= theta * rmax[r])
    S = _mk(n, n, ptr_from_rows(r[keep], n), A.col[keep].copy(), np.ones(int(keep.sum())))
    clo = from_scipy(S.sp() + S.sp().T.tocsr())
    clo = _mk(n, n, clo.ptr, clo.col, np.ones(clo.nnz))
    return S, clo


def luby_ranks(n, deg, seed):
    w = np.random.default_rng(np.random.SeedSequence(seed)).random(n) + deg / (deg + 1.0)
    order = np.lexsort((-np.arange(n), w))
    ranks = np.empty(n, dtype=I64)
    ranks[order] = np.arange(n, dtype=I64)
    return ranks


def pmisr_labels(clo, seed, max_loops=None):
    n = clo.nrows
    r = clo.rows()
    ranks = luby_ranks(n, np.diff(clo.ptr).astype(F64), seed)
    st = np.zeros(n, dtype=np.int8)       # 0 undecided, 1 fine, 2 coarse
    loops = 0
    while (st == 0).any():
        und = st == 0
        if max_loops is not None and loops >= max_loops:
            st[und] = 2
            break
        best = row_max(np.where(und[clo.col], ranks[clo.col], -1).astype(F64),
                       clo.ptr, n, empty=-1.0)
        newf = und & (ranks > best)
        st[newf] = 1
        nb = clo.col[newf[r]]
        st[nb[st[nb] == 0]] = 2
        loops += 1
    return np.where(st == 1, F_POINT, C_POINT).astype(np.int8), loops


def fsets(labels):
    return (np.flatnonzero(labels == F_POINT).astype(I64),
            np.flatnonzero(labels == C_POINT).astype(I64))


def dominance(A, labels):
    f, _ = fsets(labels)
    Aff = submatrix(A, f, f)
    d = diag_of(Aff)
    if np.any(d == 0):
        bad = f[int(np.flatnonzero(d == 0)[0])]
        raise ValueError(f'zero diagonal in fine-fine block (fine row {bad}); '
                         'splitting is not usable for reduction')
    r = Aff.rows()
    off = np.abs(np.where(Aff.col != r, Aff.val, 0.0))
    return np.bincount(r, weights=off, minlength=Aff.nrows) / np.abs(d)


def ddc(A, labels, frac, nbins):
    """One cleanup pass; returns (labels, stats dict) (splitting.py:177-207)."""
    if not 0.0 < frac < 1.0:
        raise ValueError('fraction must lie in (0, 1)')
    if nbins < 1:
        raise ValueError('nbins must be positive')
    rho = dominance(A, labels)
    nf = len(rho)
    target = frac * nf
    lo, hi = float(rho.min()), float(rho.max())
    if lo == hi:
        conv = np.full(nf, abs(nf - target) < target, dtype=bool)
        cut = lo if conv.any() else hi
    else:
        edges = lo + (hi - lo) * np.arange(nbins + 1) / nbins
        above = nf - np.searchsorted(np.sort(rho), edges, side='right')
        k = nbins - int(np.argmin(np.abs(above - target)[::-1]))
        cut = float(edges[k])
        conv = rho > cut
    f, _ = fsets(labels)
    out = labels.copy()
    out[f[conv]] = C_POINT
    return out, dict(n_f_before=nf, converted=int(conv.sum()), ratio_min=lo,
                     ratio_max=hi, ratio_mean=float(rho.mean()), cut=float(cut))


def cf_split(A, theta, frac, its, seed, nbins=1000, max_loops=None):
    _, clo = strength(A, theta)
    labels, _ = pmisr_labels(clo, seed, max_loops)
    stats = []
    for _ in range(its):
        if not (labels == F_POINT).any():
            break
        labels, s = ddc(A, labels, frac, nbins)
        stats.append(s)
    return labels, stats


# --------------------------------------------------------------------------
# polynomials (polynomial.py:40-416)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Poly:
    kind: str
    order: int
    effective_order: int
    coeffs: np.ndarray = None
    roots: np.ndarray = None
    diag_scale: np.ndarray = None
    history: tuple = None


def arnoldi(A, b, m):
    """MGS Arnoldi, one reorthogonalisation sweep when ||w|| < 0.7 ||Av||
    (polynomial.py:68-110)."""
    n = A.nrows
    m = min(m, n)
    V = np.zeros((m + 1, n))
    H = np.zeros((m + 1, m))
    beta = np.linalg.norm(b)
    if beta == 0:
        raise ValueError('cannot build a Krylov space from a zero vector')
    V[0] = b / beta
    hmax, k = 0.0, m
    for j in range(m):
        w = spmv(A, V[j])
        before = np.linalg.norm(w)
        for i in range(j + 1):
            h = V[i] @ w
            H[i, j] = h
            w -= h * V[i]
        hn = np.linalg.norm(w)
        if hn < 0.7 * before:
            for i in range(j + 1):
                h = V[i] @ w
                H[i, j] += h
                w -= h * V[i]
            hn = np.linalg.norm(w)
        H[j + 1, j] = hn
        hmax = max(hmax, np.linalg.norm(H[:j + 2, j]))
        if hn <= 1e-14 * hmax:
            H[j + 1, j] = 0.0
            k = j + 1
            break
        V[j + 1] = w / hn
    if np.max(np.abs(H[:k + 1, :k])) == 0.0:
        raise ValueError('matrix is numerically zero on the Krylov space')
    return H[:k + 1, :k], k, beta


def lsq(H, k, beta):
    rhs = np.zeros(H.shape[0])
    rhs[0] = beta
    y, *_ = np.linalg.lstsq(H[:k + 1, :k], rhs[:k + 1], rcond=None)
    return y, np.linalg.norm(rhs[:k + 1] - H[:k + 1, :k] @ y)


def arnoldi_coeffs_from_H(H, k, beta, order):
    """Monomial coefficients from the Hessenberg block (polynomial.py:148-170)."""
    hist = tuple(float(lsq(H, j, beta)[1]) for j in range(1, k + 1))
    C = np.zeros((k, k))
    C[0, 0] = 1.0
    scale = max(np.linalg.norm(H[:j + 2, j]) for j in range(k))
    powers = scale ** np.arange(k)
    growth = np.empty(k)
    growth[0] = 1.0
    for j in range(k - 1):
        sh = np.zeros(k)
        sh[1:j + 2] = C[:j + 1, j]
        C[:, j + 1] = (sh - C[:, :j + 1] @ H[:j + 1, j]) / H[j + 1, j]
        growth[j + 1] = np.abs(C[:, j + 1]) @ powers
    noise = np.finfo(np.float64).eps * np.maximum.accumulate(growth) * beta
    k_use = int(np.argmin(np.maximum(hist, noise))) + 1
    y, _ = lsq(H, k_use, beta)
    return Poly('arnoldi_coeff', order, k_use - 1, coeffs=(C[:k_use, :k_use] @ y) / beta,
                history=hist)


def gmres_poly_arnoldi(A, order, seed):
    if A.nrows != A.ncols:
        raise ValueError('require a square matrix')
    if order < 0:
        raise ValueError('order must be non-negative')
    H, k, beta = arnoldi(A, uniform_unit(A.nrows, seed), order + 1)
    return arnoldi_coeffs_from_H(H, k, beta, order)


def harmonic_ritz(H, k):
    while True:
        Hk = H[:k, :k]
        sv = np.linalg.svd(Hk, compute_uv=False)
        rank = int(np.sum(sv > 1e-12 * sv[0])) if sv[0] > 0 else 0
        if rank == 0:
            raise ValueError('matrix is numerically zero on the Krylov space')
        if rank == k:
            break
        k = rank
    hs = H[k, k - 1] if H.shape[0] > k else 0.0
    ek = np.zeros(k)
    ek[-1] = 1.0
    try:
        f = np.linalg.solve(Hk.T, ek)
    except np.linalg.LinAlgError:
        f, *_ = np.linalg.lstsq(Hk.T, ek, rcond=None)
    M = Hk.copy()
    M[:, -1] += (hs * hs) * f
    return np.linalg.eigvals(M), k


def newton_roots_from_H(H, k, beta, order, added_tol=1e-4):
    """Harmonic Ritz -> Leja-ordered units -> stability copies (polynomial.py:173-279)."""
    theta, k = harmonic_ritz(H, k)
    if np.any(np.abs(theta) == 0):
        raise ValueError('zero harmonic Ritz value; residual polynomial is degenerate')
    real = [complex(t) for t in theta[theta.imag == 0]]
    up = np.sort_complex(theta[theta.imag > 0])
    if len(up) != np.count_nonzero(theta.imag < 0):
        raise ValueError('complex roots of a real matrix must come in conjugate pairs')
    units = [(t,) for t in real] + [(t, np.conj(t)) for t in up]
    units.sort(key=lambda u: max(abs(t) for t in u), reverse=True)
    ordered = [units.pop(0)]
    placed = list(ordered[0])
    while units:
        sc = [sum(math.log(max(abs(t - p), 1e-300)) for t in u for p in placed) for u in units]
        u = units.pop(int(np.argmax(sc)))
        ordered.append(u)
        placed.extend(u)
    out, seen = [], []
    for u in ordered:
        copies = 1
        if added_tol > 0:
            for t in u:
                if any(abs(t - p) < added_tol * max(abs(t), abs(p)) for p in seen):
                    copies = 2
                    break
        for _ in range(copies):
            out.extend(u)
        seen.extend(u)
    hist = tuple(float(lsq(H, j, beta)[1]) for j in range(1, k + 1))
    return Poly('newton_roots', order, k - 1, roots=np.array(out, dtype=np.complex128),
                history=hist)


def gmres_poly_newton(A, order, seed, added_tol=1e-4):
    if A.nrows != A.ncols:
        raise ValueError('require a square matrix')
    if order < 1:
        raise ValueError('order must be at least 1')
    H, k, beta = arnoldi(A, uniform_unit(A.nrows, seed), order + 1)
    return newton_roots_from_H(H, k, beta, order, added_tol)


def neumann_poly(A, order):
    d = diag_of(A)
    if np.any(d == 0):
        raise ValueError('Neumann polynomial requires a nonzero diagonal')
    return Poly('neumann', order, order, coeffs=np.ones(order + 1), diag_scale=1.0 / d)


def apply_poly(p, A, b):
    """Matrix-free q(A) b: Horner / Neumann / factored Newton (polynomial.py:295-369)."""
    b = np.asarray(b, dtype=F64)
    if p.kind == 'arnoldi_coeff':
        c = p.coeffs
        y = c[-1] * b
        for j in range(len(c) - 2, -1, -1):
            y = spmv(A, y) + c[j] * b
        return y
    if p.kind == 'neumann':
        t = p.diag_scale * b
        acc = t.copy()
        for _ in range(p.effective_order):
            t = t - p.diag_scale * spmv(A, t)
            acc += t
        return acc
    if p.kind != 'newton_roots':
        raise ValueError(f'unknown polynomial kind {p.kind!r}')
    roots = p.roots
    x = np.zeros_like(b)
    u = b.copy()
    scale, i = 1.0, 0
    with np.errstate(over='ignore', invalid='ignore'):
        while i < len(roots):
            th = roots[i]
            if th.imag == 0:
                t = th.real
                delta = (scale / t) * u
                if not np.all(np.isfinite(delta)):
                    break
                x += delta
                u -= spmv(A, u) / t
                i += 1
            else:
                a = th.real
                m2 = (th * np.conj(th)).real
                w = spmv(A, u)
                delta = (scale / m2) * (2.0 * a * u - w)
                if not np.all(np.isfinite(delta)):
                    break
                x += delta
                u += (spmv(A, w) - 2.0 * a * w) / m2
                i += 2
            nrm = np.max(np.abs(u))
            if nrm == 0.0:
                break
            if nrm > 1e150 or nrm < 1e-150:
                u /= nrm
                scale *= nrm
                if not np.isfinite(scale) or scale == 0.0:
                    break
    return x


def assemble_poly(p, A):
    """Fixed-sparsity assembly sum_k c_k mask(A^k) (polynomial.py:372-416)."""
    if p.kind == 'newton_roots':
        raise ValueError('fixed-sparsity assembly is defined for coefficient forms only')
    n = A.nrows
    idx = np.arange(n, dtype=I64)
    pat = from_triplets(n, n, np.concatenate([A.rows(), idx]), np.concatenate([A.col, idx]),
                        np.ones(A.nnz + n))
    eye = identity(n).sp()
    if p.kind == 'arnoldi_coeff':
        base = A
    else:
        sc = _mk(n, n, A.ptr, A.col, -p.diag_scale[A.rows()] * A.val)
        base = from_scipy(eye + sc.sp())
    c = p.coeffs
    acc = c[0] * eye
    if len(c) > 1:
        acc = acc + c[1] * base.sp()
    pw = base
    for k in range(2, len(c)):
        pw = spgemm_masked(pw, base, pat)
        acc = acc + c[k] * pw.sp()
    out = from_scipy(acc)
    if p.kind == 'neumann':
        out = _mk(n, n, out.ptr, out.col, out.val * p.diag_scale[out.col])
    return out


# --------------------------------------------------------------------------
# hierarchy (hierarchy.py:55-448)
# --------------------------------------------------------------------------

ROLE_SPLIT, ROLE_SMOOTHER, ROLE_COARSE, ROLE_TRUNC_RHS = range(4)


@dataclass(frozen=True)
class Cfg:
    strong_threshold: float = 0.99
    ddc_fraction: float = 0.01
    ddc_its: int = 2
    ddc_bins: int = 1000
    poly_order: int = 6
    inverse_type: str = 'arnoldi'
    matrix_free_polys: bool = True
    a_drop: float = 1e-6
    r_drop: float = 0.0
    lump: bool = True
    coarsest_poly_order: int = 100
    coarsest_inverse_type: str = 'newton'
    auto_truncate_tol: float = 0.1
    auto_truncate_start_level: int = None
    max_levels: int = 100
    min_coarse_size: int = 16
    seed: int = 0


@dataclass
class Lvl:
    R: Csr
    P: Csr
    A_ff: Csr
    A_fc: Csr
    smoother: Poly
    labels: np.ndarray
    f: np.ndarray
    c: np.ndarray
    n: int
    nnz_A: int
    assembled: Csr = None
    A: Csr = None
    ddc_stats: list = field(default_factory=list)


@dataclass
class Hier:
    levels: list
    coarsest_A: Csr
    coarse_solver: Poly
    top_A: Csr
    truncated_at: int = None
    cycle_complexity: float = 0.0
    storage_complexity: float = 0.0
    grid_complexity: float = 0.0


def smoother_poly(A_ff, cfg, seed):
    if cfg.inverse_type == 'arnoldi':
        return gmres_poly_arnoldi(A_ff, cfg.poly_order, seed)
    return neumann_poly(A_ff, cfg.poly_order)


def coarse_poly(A, cfg, level):
    seed = derive_seed(cfg.seed, level, ROLE_COARSE)
    if cfg.coarsest_inverse_type == 'newton':
        return gmres_poly_newton(A, cfg.coarsest_poly_order, seed)
    if cfg.coarsest_inverse_type == 'arnoldi':
        return gmres_poly_arnoldi(A, cfg.coarsest_poly_order, seed)
    return neumann_poly(A, cfg.coarsest_poly_order)


def restriction(A, labels, cfg, level, smoother=None):
    """(R, A_ff, A_fc, smoother, assembled) (hierarchy.py:211-247)."""
    f, c = fsets(labels)
    A_ff, A_fc, A_cf = submatrix(A, f, f), submatrix(A, f, c), submatrix(A, c, f)
    if smoother is None:
        smoother = smoother_poly(A_ff, cfg, derive_seed(cfg.seed, level, ROLE_SMOOTHER))
    Ahat = assemble_poly(smoother, A_ff)
    Z = spgemm(A_cf, Ahat)
    Z = _mk(Z.nrows, Z.ncols, Z.ptr, Z.col, -Z.val)
    Z = drop_lump(Z, cfg.r_drop, False)
    nc = len(c)
    R = from_triplets(nc, A.nrows, np.concatenate([Z.rows(), np.arange(nc, dtype=I64)]),
                      np.concatenate([f[Z.col], c]), np.concatenate([Z.val, np.ones(nc)]))
    return R, A_ff, A_fc, smoother, Ahat


def prolongation(A, labels):
    """One-point P: first max |a_ij| over C columns (hierarchy.py:250-278)."""
    f, c = fsets(labels)
    n, nc = len(labels), len(c)
    if len(f) == 0:
        return identity(n)
    B = submatrix(A, f, c)
    lens = np.diff(B.ptr)
    if np.any(lens == 0):
        bad = f[int(np.flatnonzero(lens == 0)[0])]
        raise ValueError(f'fine point {bad} has no coupling to any coarse point; the '
                         'splitting is invalid for a one-point prolongator')
    mag = np.abs(B.val)
    mx = np.maximum.reduceat(mag, B.ptr[:-1])
    cand = np.where(mag == mx[B.rows()], np.arange(B.nnz, dtype=I64), B.nnz)
    first = np.minimum.reduceat(cand, B.ptr[:-1])
    return from_triplets(n, nc, np.concatenate([f, c]),
                         np.concatenate([B.col[first], np.arange(nc, dtype=I64)]), np.ones(n))


def galerkin(A, R, P, cfg):
    return drop_lump(spgemm(R, spgemm(A, P)), cfg.a_drop, cfg.lump)


def repair(A, labels):
    f, c = fsets(labels)
    if len(f) == 0:
        return labels
    B = submatrix(A, f, c)
    iso = np.diff(B.ptr) == 0
    if not iso.any():
        return labels
    out = labels.copy()
    out[f[iso]] = C_POINT
    return out


def truncate_start(cfg, n):
    if cfg.auto_truncate_start_level is not None:
        return cfg.auto_truncate_start_level
    reach = cfg.coarsest_poly_order + 1
    return 0 if n <= reach else int(np.ceil(np.log2(n / reach))) + 2


def truncation_test(A, cfg, level, start, solver=None):
    """(accepted solver or None, relative residual) (hierarchy.py:336-362)."""
    if cfg.auto_truncate_tol is None or level < start:
        return None, None
    if solver is None:
        try:
            solver = coarse_poly(A, cfg, level)
        except (ValueError, np.linalg.LinAlgError):
            return None, None
    rhs = uniform_unit(A.nrows, derive_seed(cfg.seed, level, ROLE_TRUNC_RHS))
    x = apply_poly(solver, A, rhs)
    res = np.linalg.norm(rhs - spmv(A, x)) / np.linalg.norm(rhs)
    if np.isfinite(res) and res <= cfg.auto_truncate_tol:
        return solver, res
    return None, res


def setup(A, cfg=Cfg(), poly_inject=None, keep_level_matrices=False):
    """Hierarchy construction (hierarchy.py:365-448).

    ``poly_inject``: optional dict with keys ``('smoother', level)`` and
    ``('coarse', level)`` mapping to ``Poly`` objects to use instead of
    recomputing them (coefficient injection).
    """
    inj = poly_inject or {}
    if A.nrows != A.ncols:
        raise ValueError('require a square matrix')
    start = truncate_start(cfg, A.nrows)
    levels, cur, lev, trunc_at, solver = [], A, 0, None, None

    def coarse_here(M, level):
        return inj.get(('coarse', level)) or coarse_poly(M, cfg, level)

    while True:
        if cur.nrows <= cfg.min_coarse_size or lev >= cfg.max_levels:
            solver = coarse_here(cur, lev)
            break
        if cfg.auto_truncate_tol is not None and lev >= start:
            cand = inj.get(('coarse', lev))
            if cand is None:
                try:
                    cand = coarse_poly(cur, cfg, lev)
                except (ValueError, np.linalg.LinAlgError):
                    cand = None
            if cand is not None:
                ok, _ = truncation_test(cur, cfg, lev, start, solver=cand)
                if ok is not None:
                    solver, trunc_at = ok, lev
                    break
        labels, stats = cf_split(cur, cfg.strong_threshold, cfg.ddc_fraction, cfg.ddc_its,
                                 derive_seed(cfg.seed, lev, ROLE_SPLIT), nbins=cfg.ddc_bins)
        nc = int((labels == C_POINT).sum())
        if nc == len(labels):
            raise ValueError(f'splitting produced no F points at level {lev}')
        if nc > 0:
            labels = repair(cur, labels)
        nf = int((labels == F_POINT).sum())
        nc = len(labels) - nf
        if nc == 0 or nf == 0:
            solver = coarse_here(cur, lev)
            break
        R, A_ff, A_fc, sm, Ahat = restriction(cur, labels, cfg, lev,
                                              smoother=inj.get(('smoother', lev)))
        P = prolongation(cur, labels)
        nxt = galerkin(cur, R, P, cfg)
        f, c = fsets(labels)
        levels.append(Lvl(R=R, P=P, A_ff=A_ff, A_fc=A_fc, smoother=sm, labels=labels, f=f, c=c,
                          n=cur.nrows, nnz_A=cur.nnz,
                          assembled=None if cfg.matrix_free_polys else Ahat,
                          A=cur if keep_level_matrices else None, ddc_stats=stats))
        cur = nxt
        lev += 1
    H = Hier(levels=levels, coarsest_A=cur, coarse_solver=solver, top_A=A, truncated_at=trunc_at)
    kept = sum(L.A_ff.nnz + L.A_fc.nnz + L.R.nnz + L.P.nnz
               + (L.assembled.nnz if L.assembled is not None else 0) for L in levels)
    H.storage_complexity = (kept + A.nnz + cur.nnz) / A.nnz
    H.cycle_complexity = cycle_flops(H) / (2.0 * A.nnz)
    H.grid_complexity = (sum(L.n for L in levels) + cur.nrows) / A.nrows
    return H


# --------------------------------------------------------------------------
# solve (solve.py:89-230)
# --------------------------------------------------------------------------


def smooth(L, rf):
    if L.assembled is not None:
        return spmv(L.assembled, rf)
    return apply_poly(L.smoother, L.A_ff, rf)


def vcycle(H, lev, r, f_smooth_its=1):
    if lev == len(H.levels):
        return apply_poly(H.coarse_solver, H.coarsest_A, r)
    L = H.levels[lev]
    ec = vcycle(H, lev + 1, spmv(L.R, r), f_smooth_its)
    rf = r[L.f]
    t = spmv(L.A_fc, ec)
    ef = smooth(L, rf - t)
    for _ in range(f_smooth_its - 1):
        ef = ef + smooth(L, rf - t - spmv(L.A_ff, ef))
    e = np.zeros(L.n)
    e[L.f] = ef
    e[L.c] = ec
    return e


class Diverged(RuntimeError):
    def __init__(self, msg, iteration):
        super().__init__(msg)
        self.iteration = iteration


def richardson(H, b, x0, rtol=1e-10, atol=1e-50, max_iters=100, f_smooth_its=1):
    A = H.top_A
    b = np.asarray(b, dtype=F64)
    x = np.array(x0, dtype=F64, copy=True)
    r = b - spmv(A, x)
    rn = float(np.linalg.norm(r))
    hist = [rn]
    bn = float(np.linalg.norm(b))
    thr = max(rtol * (bn if bn > 0 else rn), atol)
    if not np.isfinite(rn):
        raise Diverged('non-finite residual at iteration 0', 0)
    conv, its = rn <= thr, 0
    while not conv and its < max_iters:
        x += vcycle(H, 0, r, f_smooth_its)
        r = b - spmv(A, x)
        rn = float(np.linalg.norm(r))
        its += 1
        hist.append(rn)
        if not np.isfinite(rn):
            raise Diverged(f'non-finite residual at iteration {its}', its)
        if rn > 1e8 * hist[0]:
            raise Diverged(f'residual grew by more than 1e+08 at iteration {its}', its)
        conv = rn <= thr
    return x, hist, conv, its


def poly_flops(p, nnz, n):
    if p.kind == 'arnoldi_coeff':
        return 2 * n + (len(p.coeffs) - 1) * (2 * nnz + 2 * n)
    if p.kind == 'neumann':
        return 2 * n + p.effective_order * (2 * nnz + 6 * n)
    tot, i = 0, 0
    while i < len(p.roots):
        if p.roots[i].imag == 0:
            tot += 2 * nnz + 4 * n
            i += 1
        else:
            tot += 4 * nnz + 10 * n
            i += 2
    return tot


def cycle_flops(H, f_smooth_its=1):
    tot = 0
    for L in H.levels:
        nf = len(L.f)
        sm = 2 * L.assembled.nnz if L.assembled is not None else poly_flops(L.smoother, L.A_ff.nnz, nf)
        tot += 2 * L.R.nnz + 2 * L.A_fc.nnz + 2 * nf + sm
        tot += (f_smooth_its - 1) * (2 * L.A_ff.nnz + 4 * nf + sm + 2 * nf)
    return int(tot + poly_flops(H.coarse_solver, H.coarsest_A.nnz, H.coarsest_A.nrows))


def cycle_bytes(H):
    """Algorithmic HBM bytes of one V-cycle + top residual."""
    def spm(M):
        return 12 * M.nnz + 4 * (M.nrows + 1)
    tot = 0
    for L in H.levels:
        nf, nc = len(L.f), len(L.c)
        d = len(L.smoother.coeffs) - 1 if L.smoother.coeffs is not None else 0
        tot += spm(L.R) + 8 * L.n + 8 * nc
        tot += spm(L.A_fc) + 8 * nc + 16 * nf
        tot += 16 * nf + d * (spm(L.A_ff) + 24 * nf)
        tot += 16 * L.n
    C = H.coarsest_A
    p = H.coarse_solver
    if p.kind == 'newton_roots':
        i = 0
        while i < len(p.roots):
            if p.roots[i].imag == 0:
                tot += spm(C) + 32 * C.nrows
                i += 1
            else:
                tot += 2 * spm(C) + 56 * C.nrows
                i += 2
    else:
        tot += 16 * C.nrows + (len(p.coeffs) - 1) * (spm(C) + 24 * C.nrows)
    tot += spm(H.top_A) + 40 * H.top_A.nrows
    return int(tot)
