"""V-cycle and Richardson outer iteration on the GPU (ref: solve.py:19-230).

The hierarchy's operators stay in HBM; a native plan (``airg_plan`` in
libairg.so) holds their device pointers and issues the whole V-cycle --
restriction SpMVs, the single-CTA Newton coarse solve, fused
``r_f - A_fc e_c`` residuals, Horner smoothing chains and the scatters --
from C++, so Python is off the per-cycle path.
"""

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .csr import VAL, empty, is_host_array, to_dev
from .gmres_poly import poly_args

_DIVERGENCE_FACTOR = 1e8


@dataclass(frozen=True)
class SolveConfig:
    """Outer-iteration controls (solve.py:31-54)."""

    rtol: float = 1e-10
    atol: float = 1e-50
    max_iters: int = 100
    f_smooth_its: int = 1

    def validate(self):
        if self.rtol <= 0:
            raise ValueError('rtol must be positive')
        if self.atol < 0:
            raise ValueError('atol must be non-negative')
        if self.max_iters < 1:
            raise ValueError('max_iters must be at least 1')
        if self.f_smooth_its < 1:
            raise ValueError('f_smooth_its must be at least 1')
        return self


@dataclass
class SolveStats:
    """Iteration record (solve.py:57-77)."""

    iterations: int
    residual_history: list
    converged: bool
    cycle_complexity: float
    storage_complexity: float
    flops_per_cycle: int

    def to_dict(self):
        return {
            'iterations': self.iterations,
            'residual_history': [float(r) for r in self.residual_history],
            'converged': self.converged,
            'cycle_complexity': self.cycle_complexity,
            'storage_complexity': self.storage_complexity,
            'flops_per_cycle': self.flops_per_cycle,
        }


class DivergenceError(RuntimeError):
    """Non-finite or exploding outer residual (solve.py:80-86)."""

    def __init__(self, message, iteration):
        super().__init__(message)
        self.iteration = iteration


class Plan:
    """Owner of a native ``airg_plan`` built from a Hierarchy."""

    def __init__(self, H):
        self.h = C.c_void_p()
        L.call('airg_plan_create', len(H.levels), C.byref(self.h))
        self._keep = []
        A = H.top_A
        L.call('airg_plan_set_top', self.h, A.nrows, L.ptr(A.row_offsets), L.ptr(A.col_indices),
               L.ptr(A.values))
        for i, lv in enumerate(H.levels):
            code, nc, c, nu, t, a1, a2, ds, keep = poly_args(lv.f_smoother)
            if code == 1:
                raise ValueError('Newton-form fine smoothers are not supported')
            asm = lv.f_smoother_assembled
            L.call('airg_plan_set_level', self.h, i, lv.n, lv.split.n_f, lv.split.n_c,
                   L.ptr(lv.R.row_offsets), L.ptr(lv.R.col_indices), L.ptr(lv.R.values),
                   L.ptr(lv.A_fc.row_offsets), L.ptr(lv.A_fc.col_indices), L.ptr(lv.A_fc.values),
                   L.ptr(lv.A_ff.row_offsets), L.ptr(lv.A_ff.col_indices), L.ptr(lv.A_ff.values),
                   L.ptr(lv.split.f_idx), L.ptr(lv.split.c_idx), code, nc, L.hptr(c), L.ptr(ds),
                   -1 if asm is None else asm.nnz,
                   None if asm is None else L.ptr(asm.row_offsets),
                   None if asm is None else L.ptr(asm.col_indices),
                   None if asm is None else L.ptr(asm.values))
        Cm = H.coarsest_A
        code, nc, c, nu, t, a1, a2, ds, keep = poly_args(H.coarse_solver)
        L.call('airg_plan_set_coarse', self.h, Cm.nrows, L.ptr(Cm.row_offsets),
               L.ptr(Cm.col_indices), L.ptr(Cm.values), code, nc, L.hptr(c), nu, L.hptr(t),
               L.hptr(a1), L.hptr(a2), L.ptr(ds))
        # The plan is owned by H (H._plan) and H owns every device buffer the
        # plan points at; no back-reference, so dropping H frees both at once
        # (a cycle here left whole hierarchies to the cyclic GC).

    def __del__(self):
        try:
            if self.h:
                L.load().airg_plan_destroy(self.h)
        except Exception:
            pass

    def launches(self):
        return int(L.load().airg_plan_launches(self.h))


class _PlanPool:
    """Native plans of one Hierarchy, one per concurrent solve.

    The reference's Hierarchy is immutable and usable by concurrent solves,
    each owning its work vectors (SPEC.md concurrency model, solve.py:113-167).
    A plan holds work vectors, a stream and its captured graphs, so a solve
    takes a plan from the pool for its whole duration (creating one when all
    are busy) and returns it afterwards; the arithmetic mode is set on the
    taken plan, never on a shared one."""

    def __init__(self):
        import threading
        self.lock = threading.Lock()
        self.free = []
        self.all = []

    def acquire(self, H, exact):
        with self.lock:
            p = self.free.pop() if self.free else None
        if p is None:
            p = Plan(H)
            with self.lock:
                self.all.append(p)
        L.call('airg_plan_set_exact', p.h, 1 if exact else 0)
        return p

    def release(self, p):
        with self.lock:
            self.free.append(p)


_POOL_LOCK = None


def _pool(H):
    global _POOL_LOCK
    pool = H.__dict__.get('_plans')
    if pool is None:
        import threading
        if _POOL_LOCK is None:
            _POOL_LOCK = threading.Lock()
        with _POOL_LOCK:
            pool = H.__dict__.get('_plans')
            if pool is None:
                pool = _PlanPool()
                H._plans = pool
    return pool


class plan_for:
    """Context manager: ``with plan_for(H, exact) as p`` holds a plan of H's
    pool for the duration of one solve."""

    def __init__(self, H, exact=False):
        self.H, self.exact = H, exact

    def __enter__(self):
        self.p = _pool(self.H).acquire(self.H, self.exact)
        return self.p

    def __exit__(self, *exc):
        _pool(self.H).release(self.p)
        return False


def held_plan(H, exact=False):
    """A plan of H's pool taken for good (measurement tools that drive the
    native plan directly)."""
    return _pool(H).acquire(H, exact)


def coarse_mode(H):
    """'dense' when the fast-mode coarse solve of H's plans is the dense q(A)
    GEMV, 'newton' otherwise (after a solve has built a plan)."""
    pool = H.__dict__.get('_plans')
    if pool is None or not pool.all:
        return None
    return 'dense' if L.load().airg_plan_coarse_mode(pool.all[0].h) == 1 else 'newton'


def _level_size(H, level):
    if level == len(H.levels):
        return H.coarsest_A.nrows
    return H.levels[level].n


def vcycle(H, level, r, cfg, exact=False):
    """Error estimate for A_level e = r from one V-cycle (solve.py:95-110).
    ``exact=True`` runs the reference-order arithmetic (parity mode)."""
    if level < 0 or level > len(H.levels):
        raise ValueError(f'level {level} out of range')
    n = _level_size(H, level)
    host = is_host_array(r)
    r = to_dev(r, VAL)
    if r.numel() != n:
        raise ValueError('residual has wrong length for this level')
    e = empty(n, VAL)
    with plan_for(H, exact) as p:
        L.call('airg_plan_vcycle', p.h, level, L.ptr(r), L.ptr(e), cfg.f_smooth_its,
               L.stream_handle())
    return e.cpu().numpy() if host else e


def richardson_solve(H, b, x0, cfg, exact=False):
    """Undamped Richardson iteration preconditioned by one V-cycle
    (solve.py:113-167).  ``b``/``x0`` may be numpy or device tensors; ``x`` is
    returned as a device tensor.  ``exact=True`` selects the parity mode in
    which every kernel follows the reference's arithmetic order (x is then
    bitwise the reference's for the same hierarchy); the default is the fast
    vector/FMA path."""
    cfg.validate()
    A = H.top_A
    host = is_host_array(x0)
    b = to_dev(b, VAL)
    x = to_dev(x0, VAL).clone()
    if b.numel() != A.nrows or x.numel() != A.nrows:
        raise ValueError('right-hand side or initial guess has wrong length')
    hist = np.zeros(cfg.max_iters + 1)
    its = C.c_int(0)
    conv = C.c_int(0)
    with plan_for(H, exact) as plan:
        st = L.load().airg_plan_richardson(plan.h, L.ptr(b), L.ptr(x), cfg.rtol, cfg.atol,
                                           cfg.max_iters, cfg.f_smooth_its, L.hptr(hist),
                                           C.byref(its), C.byref(conv), L.stream_handle())
    if st == L.ERR_DIVERGED:
        raise DivergenceError(L.last_error(), its.value)
    L.check(st, 'airg_plan_richardson')
    stats = SolveStats(iterations=its.value, residual_history=list(hist[:its.value + 1]),
                       converged=bool(conv.value), cycle_complexity=H.cycle_complexity,
                       storage_complexity=H.storage_complexity,
                       flops_per_cycle=count_cycle_flops(H, f_smooth_its=cfg.f_smooth_its))
    # the reference returns an ndarray: numpy in, numpy out; device in, device out
    return (x.cpu().numpy() if host else x), stats


def _poly_apply_flops(p, nnz, n):
    if p.kind == 'arnoldi_coeff':
        return 2 * n + (len(p.coeffs) - 1) * (2 * nnz + 2 * n)
    if p.kind == 'neumann':
        return 2 * n + p.effective_order * (2 * nnz + 6 * n)
    if p.kind == 'newton_roots':
        tot, i = 0, 0
        while i < len(p.roots):
            if p.roots[i].imag == 0:
                tot += 2 * nnz + 4 * n
                i += 1
            else:
                tot += 4 * nnz + 10 * n
                i += 2
        return tot
    raise ValueError(f'unknown polynomial kind {p.kind!r}')


def count_cycle_flops(H, f_smooth_its=1):
    """Deterministic FLOP model of one V-cycle (solve.py:170-230)."""
    tot = 0
    for lv in H.levels:
        nf = lv.split.n_f
        if lv.f_smoother_assembled is not None:
            sm = 2 * lv.f_smoother_assembled.nnz
        else:
            sm = _poly_apply_flops(lv.f_smoother, lv.A_ff.nnz, nf)
        tot += 2 * lv.R.nnz + 2 * lv.A_fc.nnz + 2 * nf + sm
        tot += (f_smooth_its - 1) * (2 * lv.A_ff.nnz + 4 * nf + sm + 2 * nf)
    tot += _poly_apply_flops(H.coarse_solver, H.coarsest_A.nnz, H.coarsest_A.nrows)
    return int(tot)


def _spmat_bytes(M):
    return 12 * M.nnz + 4 * (M.nrows + 1)


def count_cycle_bytes(H, include_top=True, coarse=None):
    """Algorithmic HBM bytes of one V-cycle (+ the top residual), the
    roofline numerator of SURVEY.md 8(d): 12 B/nnz + 4 B/row per matrix pass,
    every vector operand read or written once.  ``coarse``: the coarse solve
    that runs -- 'dense' (fast mode's q(A) GEMV: 8 n^2 + 16 n) or 'newton'
    (the root-by-root apply); default: what H's solve plans use."""
    if coarse is None:
        coarse = coarse_mode(H) or 'newton'
    tot = 0
    for lv in H.levels:
        nf, nc = lv.split.n_f, lv.split.n_c
        p = lv.f_smoother
        d = len(p.coeffs) - 1 if p.coeffs is not None else 0
        tot += _spmat_bytes(lv.R) + 8 * lv.n + 8 * nc
        if (lv.f_smoother_assembled is None and p.kind == 'arnoldi_coeff' and d == 0
                and lv.A_fc.nrows > 0):
            # fused: e[f] = c0 (r[f] - A_fc e_c) and the e[c] scatter in one pass
            tot += _spmat_bytes(lv.A_fc) + 24 * nc + 16 * nf
            continue
        tot += _spmat_bytes(lv.A_fc) + 8 * nc + 16 * nf
        if lv.f_smoother_assembled is not None:
            tot += 16 * nf + _spmat_bytes(lv.f_smoother_assembled)
            tot += 16 * lv.n                      # scatter e[f] = e_f, e[c] = e_c
        else:
            tot += 16 * nf + d * (_spmat_bytes(lv.A_ff) + 24 * nf)
            if p.kind == 'arnoldi_coeff' and d > 0:
                tot += 16 * nc                    # e[f] written by the last Horner step
            else:
                tot += 16 * lv.n
    Cm, p = H.coarsest_A, H.coarse_solver
    if p.kind == 'newton_roots' and coarse == 'dense':
        tot += 8 * Cm.nrows * Cm.nrows + 16 * Cm.nrows
    elif p.kind == 'newton_roots':
        i = 0
        while i < len(p.roots):
            if p.roots[i].imag == 0:
                tot += _spmat_bytes(Cm) + 32 * Cm.nrows
                i += 1
            else:
                tot += 2 * _spmat_bytes(Cm) + 56 * Cm.nrows
                i += 2
    else:
        tot += 16 * Cm.nrows + (len(p.coeffs) - 1) * (_spmat_bytes(Cm) + 24 * Cm.nrows)
    if include_top:
        tot += _spmat_bytes(H.top_A) + 40 * H.top_A.nrows
    return int(tot)
