"""GMRES polynomial approximate inverses (ref: polynomial.py:25-431).

The Krylov basis (SpMVs, MGS dot products, norms) is built on the GPU; the
(order+2) x (order+1) Hessenberg block comes back to the host, where the
O(m^3) dense algebra (least squares, SVD, eigenvalues, Leja ordering) runs in
numpy -- the control plane, exactly the routines the reference calls.
Application (Horner / factored Newton / Neumann) is a device kernel chain.
"""

import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .csr import VAL, empty, to_dev

KIND_CODE = {'arnoldi_coeff': 0, 'newton_roots': 1, 'neumann': 2}


@dataclass(frozen=True)
class PolySolver:
    """Fixed polynomial approximation of a matrix inverse (polynomial.py:40-58)."""

    kind: str
    order: int
    effective_order: int
    coeffs: np.ndarray = None
    roots: np.ndarray = None
    diag_scale: object = None       # device fp64 tensor (neumann)
    residual_history: tuple = None


def newton_units(roots):
    """Encode Leja-ordered roots as units: real theta -> (0, theta, 0); a
    conjugate pair (a +- bi) -> (1, 2a, |theta|^2) (polynomial.py:324-345)."""
    types, p1, p2 = [], [], []
    i = 0
    while i < len(roots):
        th = roots[i]
        if th.imag == 0:
            types.append(0)
            p1.append(th.real)
            p2.append(0.0)
            i += 1
        else:
            types.append(1)
            p1.append(2.0 * th.real)
            p2.append((th * np.conj(th)).real)
            i += 2
    return (np.array(types, dtype=np.int32), np.array(p1, dtype=np.float64),
            np.array(p2, dtype=np.float64))


def poly_args(p):
    """(kind, ncoef, coef_h, nunits, type_h, p1_h, p2_h, diag_scale_tensor, keepalive)."""
    code = KIND_CODE.get(p.kind)
    if code is None:
        raise ValueError(f'unknown polynomial kind {p.kind!r}')
    if code == 1:
        t, a, b = newton_units(p.roots)
        return code, 0, None, len(t), t, a, b, None, (t, a, b)
    c = np.ascontiguousarray(p.coeffs, dtype=np.float64)
    ds = p.diag_scale if code == 2 else None
    return code, len(c), c, 0, None, None, None, ds, (c,)


def apply_matrix_free(p, A, b, exact=False):
    """q(A) b with SpMVs and vector updates only (polynomial.py:358-369).
    ``exact=True`` follows the reference's arithmetic order bit for bit."""
    if p.kind not in KIND_CODE:
        raise ValueError(f'unknown polynomial kind {p.kind!r}')
    b = to_dev(b, VAL)
    if A.nrows != A.ncols or b.numel() != A.ncols:
        raise ValueError('solver, matrix and vector shapes disagree')
    code, nc, c, nu, t, a1, a2, ds, keep = poly_args(p)
    y = empty(A.nrows, VAL)
    L.call('airg_poly_apply', code, A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices),
           L.ptr(A.values), nc, L.hptr(c), nu, L.hptr(t), L.hptr(a1), L.hptr(a2), L.ptr(ds),
           L.ptr(b), L.ptr(y), 1 if exact else 0, L.stream_handle())
    del keep
    return y


# ---------------------------------------------------------------------------
# host-side dense algebra on the device-built Hessenberg block
# ---------------------------------------------------------------------------

_BLAS_CTL = None


def _one_blas_thread():
    """Context limiting BLAS to one thread: the Hessenberg blocks are at most
    102 x 101, where a multi-threaded OpenBLAS spends far longer waking and
    synchronising its pool than computing (eigvals of 100 x 100: 311 ms on 8
    threads vs 13 ms on one, measured)."""
    global _BLAS_CTL
    try:
        if _BLAS_CTL is None:
            from threadpoolctl import ThreadpoolController
            _BLAS_CTL = ThreadpoolController()
        return _BLAS_CTL.limit(limits=1, user_api='blas')
    except Exception:  # threadpoolctl missing: run as is
        import contextlib
        return contextlib.nullcontext()

def _lsq(H, k, beta):
    rhs = np.zeros(H.shape[0])
    rhs[0] = beta
    y, *_ = np.linalg.lstsq(H[:k + 1, :k], rhs[:k + 1], rcond=None)
    return y, np.linalg.norm(rhs[:k + 1] - H[:k + 1, :k] @ y)


def _history(H, k, beta):
    return tuple(float(_lsq(H, j, beta)[1]) for j in range(1, k + 1))


def coeffs_from_hessenberg(H, k, beta, order):
    """Monomial GMRES-polynomial coefficients with the noise-limited order
    choice (polynomial.py:148-170)."""
    with _one_blas_thread():
        return _coeffs_from_hessenberg(H, k, beta, order)


def _coeffs_from_hessenberg(H, k, beta, order):
    hist = _history(H, k, beta)
    Cb = np.zeros((k, k))
    Cb[0, 0] = 1.0
    scale = max(np.linalg.norm(H[:j + 2, j]) for j in range(k))
    powers = scale ** np.arange(k)
    growth = np.empty(k)
    growth[0] = 1.0
    for j in range(k - 1):
        sh = np.zeros(k)
        sh[1:j + 2] = Cb[:j + 1, j]
        Cb[:, j + 1] = (sh - Cb[:, :j + 1] @ H[:j + 1, j]) / H[j + 1, j]
        growth[j + 1] = np.abs(Cb[:, j + 1]) @ powers
    noise = np.finfo(np.float64).eps * np.maximum.accumulate(growth) * beta
    k_use = int(np.argmin(np.maximum(hist, noise))) + 1
    y, _ = _lsq(H, k_use, beta)
    return PolySolver('arnoldi_coeff', order, k_use - 1, coeffs=(Cb[:k_use, :k_use] @ y) / beta,
                      residual_history=hist)


def roots_from_hessenberg(H, k, beta, order, added_root_tol=1e-4):
    """Harmonic Ritz values, Leja order, stability copies (polynomial.py:173-279)."""
    with _one_blas_thread():
        return _roots_from_hessenberg(H, k, beta, order, added_root_tol)


def _roots_from_hessenberg(H, k, beta, order, added_root_tol):
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
    theta = np.linalg.eigvals(M)
    if np.any(np.abs(theta) == 0):
        raise ValueError('zero harmonic Ritz value; residual polynomial is degenerate')
    real = [complex(t) for t in theta[theta.imag == 0]]
    upper = np.sort_complex(theta[theta.imag > 0])
    if len(upper) != np.count_nonzero(theta.imag < 0):
        raise ValueError('complex roots of a real matrix must come in conjugate pairs')
    pool = [(t,) for t in real] + [(t, np.conj(t)) for t in upper]
    pool.sort(key=lambda u: max(abs(t) for t in u), reverse=True)
    # Leja order by summed log-distance to the placed roots; the score of each
    # remaining unit is updated incrementally (O(m^2) numpy instead of the
    # reference's O(m^3) Python loop; ties still go to the first unit).
    first = np.array([u[0] for u in pool], dtype=np.complex128)
    second = np.array([u[1] if len(u) > 1 else np.nan for u in pool], dtype=np.complex128)
    is_pair = np.array([len(u) > 1 for u in pool])
    alive = np.ones(len(pool), dtype=bool)
    score = np.zeros(len(pool))

    def place(i):
        alive[i] = False
        for q in pool[i]:
            d = np.log(np.maximum(np.abs(first - q), 1e-300))
            d2 = np.where(is_pair, np.log(np.maximum(np.abs(second - q), 1e-300)), 0.0)
            score[:] += d + d2

    seq = [pool[0]]
    place(0)
    while alive.any():
        cand = np.flatnonzero(alive)
        i = int(cand[np.argmax(score[cand])])
        seq.append(pool[i])
        place(i)
    # stability copies: a unit is doubled when one of its roots lies within
    # the relative gap of an earlier root (same comparisons, vectorised over
    # the placed roots)
    out = []
    seen = np.empty(sum(len(u) for u in seq), dtype=np.complex128)
    ns = 0
    for u in seq:
        reps = 1
        if added_root_tol > 0 and ns:
            s_ = seen[:ns]
            as_ = np.abs(s_)
            for t in u:
                if np.any(np.abs(t - s_) < added_root_tol * np.maximum(abs(t), as_)):
                    reps = 2
                    break
        for _ in range(reps):
            out.extend(u)
        seen[ns:ns + len(u)] = u
        ns += len(u)
    return PolySolver('newton_roots', order, k - 1, roots=np.array(out, dtype=np.complex128),
                      residual_history=_history_givens(H, k, beta))


def _history_givens(H, k, beta):
    """GMRES residual norms for steps 1..k from one Givens QR sweep of the
    Hessenberg block (diagnostic history of the Newton kind; O(k^2) instead
    of k least-squares solves)."""
    R = np.array(H[:k + 1, :k], dtype=np.float64, copy=True)
    g = np.zeros(k + 1)
    g[0] = beta
    out = []
    for j in range(k):
        a, b = R[j, j], R[j + 1, j]
        r = math.hypot(a, b)
        c, s = (1.0, 0.0) if r == 0 else (a / r, b / r)
        Rj, Rj1 = R[j, j:].copy(), R[j + 1, j:].copy()
        R[j, j:] = c * Rj + s * Rj1
        R[j + 1, j:] = -s * Rj + c * Rj1
        g[j], g[j + 1] = c * g[j], -s * g[j]
        out.append(float(abs(g[j + 1])))
    return tuple(out)


def hessenberg(A, m, b):
    """Device Arnoldi (polynomial.py:68-110): returns (H (m+1) x m, k, beta)."""
    import ctypes as C
    n = A.nrows
    m = min(m, n)
    H = np.zeros((m + 1, m))
    k = C.c_int32()
    beta = C.c_double()
    L.call('airg_arnoldi', n, L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
           L.ptr(b), m, L.hptr(H), C.byref(k), C.byref(beta), L.stream_handle())
    k = k.value
    return H[:k + 1, :k].copy(), k, beta.value


def gmres_poly_arnoldi(A, order, seed):
    """Minimum-residual polynomial in monomial form (polynomial.py:126-170)."""
    from .csr import random_unit_vector
    if A.nrows != A.ncols:
        raise ValueError('require a square matrix')
    if order < 0:
        raise ValueError('order must be non-negative')
    b = random_unit_vector(A.nrows, seed)
    H, k, beta = hessenberg(A, order + 1, b)
    return coeffs_from_hessenberg(H, k, beta, order)


def gmres_poly_newton(A, order, seed, added_root_tol=1e-4):
    """Minimum-residual polynomial in factored Newton form (polynomial.py:257-279)."""
    from .csr import random_unit_vector
    if A.nrows != A.ncols:
        raise ValueError('require a square matrix')
    if order < 1:
        raise ValueError('order must be at least 1')
    b = random_unit_vector(A.nrows, seed)
    H, k, beta = hessenberg(A, order + 1, b)
    return roots_from_hessenberg(H, k, beta, order, added_root_tol)


def neumann_poly(A, order):
    """Truncated Neumann series sum_k (I - D^-1 A)^k D^-1 (polynomial.py:282-292)."""
    from .csr import diagonal
    if A.nrows != A.ncols:
        raise ValueError('require a square matrix')
    if order < 0:
        raise ValueError('order must be non-negative')
    d = diagonal(A)
    if bool((d == 0).any()):
        raise ValueError('Neumann polynomial requires a nonzero diagonal')
    return PolySolver('neumann', order, order, coeffs=np.ones(order + 1), diag_scale=1.0 / d)


def assemble_fixed_sparsity(p, A):
    """sum_k c_k mask(A^k), mask = pattern(A) + diagonal (polynomial.py:372-416)."""
    import ctypes as C
    from .csr import take
    if p.kind == 'newton_roots':
        raise ValueError('fixed-sparsity assembly is defined for coefficient forms only, not '
                         'newton_roots')
    if A.nrows != A.ncols:
        raise ValueError('require a square matrix')
    if p.kind not in ('arnoldi_coeff', 'neumann'):
        raise ValueError(f'unknown polynomial kind {p.kind!r}')
    c = np.ascontiguousarray(p.coeffs, dtype=np.float64)
    base = A
    if p.kind == 'neumann':
        # series in N = I - D^-1 A (zeros pruned), mask from A itself
        rb = C.c_void_p()
        L.call('airg_neumann_base', A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices),
               L.ptr(A.values), L.ptr(p.diag_scale), C.byref(rb), L.stream_handle())
        base = take(rb)
    r = C.c_void_p()
    L.call('airg_poly_assemble', A.nrows, L.ptr(base.row_offsets), L.ptr(base.col_indices),
           L.ptr(base.values), len(c), L.hptr(c), L.ptr(A.row_offsets), L.ptr(A.col_indices),
           C.byref(r), L.stream_handle())
    out = take(r)
    if p.kind == 'neumann':
        L.call('airg_scale_columns', out.nnz, L.ptr(out.col_indices), L.ptr(p.diag_scale),
               L.ptr(out.values), L.stream_handle())
    return out


def export_diagnostics(p):
    """JSON-serialisable description (polynomial.py:419-431)."""
    return {
        'kind': p.kind,
        'order': p.order,
        'effective_order': p.effective_order,
        'coeffs': None if p.coeffs is None else [float(c) for c in p.coeffs],
        'roots': None if p.roots is None else [[float(r.real), float(r.imag)] for r in p.roots],
        'generating_residual_history':
            None if p.residual_history is None else list(p.residual_history),
    }
