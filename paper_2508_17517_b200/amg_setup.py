"""Multigrid hierarchy construction on the GPU (ref: hierarchy.py:27-490).

Per level: (truncation test) -> CF splitting -> restriction / prolongation ->
Galerkin coarse matrix R (A P) with drop/lump, every step an sm_100a kernel in
libairg.so; only the tiny dense Krylov algebra runs on the host.
"""

import logging
import time
from dataclasses import dataclass, field, fields

import numpy as np

_log = logging.getLogger(__name__)

SEED_SPLIT, SEED_SMOOTHER, SEED_COARSE_POLY, SEED_TRUNC_RHS = range(4)

SETUP_PHASES = ('cf_split', 'prolongator', 'polynomial', 'spgemm_R', 'spgemm_coarse', 'extract',
                'drop', 'truncation')

_INVERSE_TYPES = ('arnoldi', 'neumann')
_COARSEST_INVERSE_TYPES = ('newton', 'arnoldi', 'neumann')


def derive_seed(root, level, role):
    """SeedSequence([root, level, role]) -> uint32 (hierarchy.py:50-52)."""
    return int(np.random.SeedSequence([root, level, role]).generate_state(1)[0])


@dataclass(frozen=True)
class SetupConfig:
    """Hierarchy construction parameters (hierarchy.py:55-138)."""

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
    smooth_type: str = 'f'
    one_point_classical_prolong: bool = True
    improve_z_its: int = 0
    improve_w_its: int = 0
    inverse_sparsity_order: int = 1

    def validate(self):
        if not 0.0 <= self.strong_threshold <= 1.0:
            raise ValueError('strong_threshold must lie in [0, 1]')
        if not 0.0 < self.ddc_fraction < 1.0:
            raise ValueError('ddc_fraction must lie in (0, 1)')
        if self.ddc_its < 0:
            raise ValueError('ddc_its must be non-negative')
        if self.ddc_bins < 1:
            raise ValueError('ddc_bins must be positive')
        if self.poly_order < 0:
            raise ValueError('poly_order must be non-negative')
        if self.inverse_type not in _INVERSE_TYPES:
            raise ValueError(f'inverse_type must be one of {_INVERSE_TYPES}')
        if self.a_drop < 0 or self.r_drop < 0:
            raise ValueError('drop tolerances must be non-negative')
        if self.coarsest_inverse_type not in _COARSEST_INVERSE_TYPES:
            raise ValueError(f'coarsest_inverse_type must be one of {_COARSEST_INVERSE_TYPES}')
        min_order = 1 if self.coarsest_inverse_type == 'newton' else 0
        if self.coarsest_poly_order < min_order:
            raise ValueError(f'coarsest_poly_order too small for {self.coarsest_inverse_type}')
        if self.auto_truncate_tol is not None and self.auto_truncate_tol < 0:
            raise ValueError('auto_truncate_tol must be non-negative or None')
        if self.auto_truncate_start_level is not None and self.auto_truncate_start_level < 0:
            raise ValueError('auto_truncate_start_level must be non-negative or None for the '
                             'a priori estimate')
        if self.max_levels < 1:
            raise ValueError('max_levels must be at least 1')
        if self.min_coarse_size < 1:
            raise ValueError('min_coarse_size must be at least 1')
        if self.seed < 0:
            raise ValueError('seed must be non-negative')
        if self.smooth_type != 'f':
            raise ValueError("only fine-point smoothing is supported (smooth_type='f'); C-point "
                             'and FCF smoothing are not implemented')
        if not self.one_point_classical_prolong:
            raise ValueError('approximate ideal prolongation is not implemented; only the '
                             'one-point classical prolongator is supported')
        if self.improve_z_its != 0 or self.improve_w_its != 0:
            raise ValueError('Richardson improvement of the transfer operators is not '
                             'implemented')
        if self.inverse_sparsity_order != 1:
            raise ValueError('only inverse_sparsity_order=1 is implemented')
        return self

    def to_dict(self):
        return {f.name: getattr(self, f.name) for f in fields(self)}


@dataclass
class Level:
    """Operators retained for the solve on one level (hierarchy.py:141-160)."""

    R: object
    P: object
    A_ff: object
    A_fc: object
    f_smoother: object
    split: object
    n: int
    nnz_A: int
    f_smoother_assembled: object = None
    ddc_stats: tuple = ()


@dataclass
class Hierarchy:
    """Per-level operators + coarsest matrix and solver (hierarchy.py:163-181)."""

    levels: list
    coarsest_A: object
    coarse_solver: object
    top_A: object
    cycle_complexity: float = 0.0
    storage_complexity: float = 0.0
    grid_complexity: float = 0.0
    truncated_at: int = None
    config: SetupConfig = None
    setup_breakdown: dict = field(default_factory=dict)

    @property
    def num_levels(self):
        return len(self.levels)


def finalize_complexities(H):
    """Storage / cycle / grid complexity (hierarchy.py:439-447)."""
    from .amg_solve import count_cycle_flops
    A = H.top_A
    kept = 0
    for lv in H.levels:
        kept += lv.A_ff.nnz + lv.A_fc.nnz + lv.R.nnz + lv.P.nnz
        if lv.f_smoother_assembled is not None:
            kept += lv.f_smoother_assembled.nnz
    H.storage_complexity = (kept + A.nnz + H.coarsest_A.nnz) / A.nnz
    H.cycle_complexity = count_cycle_flops(H) / (2.0 * A.nnz)
    H.grid_complexity = (sum(lv.n for lv in H.levels) + H.coarsest_A.nrows) / A.nrows
    return H


def setup_compulsory_bytes(H):
    """Compulsory HBM traffic of the setup: every level operator read once
    and every retained output (R, P, A_ff, A_fc and the next level's
    operator) written once, 12 B/nnz + 4 B/row (int32 CSR, fp64 values).
    Intermediates (Z, A P, the assembled polynomial, pre-drop R A P rows)
    are not counted: this is the lower bound a memory-bound setup would
    approach, not the bytes the kernels move."""
    def spm(nnz, rows):
        return 12 * int(nnz) + 4 * (int(rows) + 1)
    tot = 0
    for i, lv in enumerate(H.levels):
        nxt = H.levels[i + 1] if i + 1 < len(H.levels) else None
        tot += spm(lv.nnz_A, lv.n)
        for M in (lv.R, lv.P, lv.A_ff, lv.A_fc):
            tot += spm(M.nnz, M.nrows)
        tot += spm(nxt.nnz_A, nxt.n) if nxt is not None else spm(H.coarsest_A.nnz,
                                                                  H.coarsest_A.nrows)
    if not H.levels:
        tot += spm(H.top_A.nnz, H.top_A.nrows)
    return int(tot)


def hierarchy_summary(H):
    """JSON-serialisable summary (hierarchy.py:451-490)."""
    levels = []
    for idx, lv in enumerate(H.levels):
        levels.append({
            'level': idx, 'n': int(lv.n), 'n_f': int(lv.split.n_f), 'n_c': int(lv.split.n_c),
            'nnz_A': int(lv.nnz_A), 'nnz_A_ff': int(lv.A_ff.nnz), 'nnz_A_fc': int(lv.A_fc.nnz),
            'nnz_R': int(lv.R.nnz), 'nnz_P': int(lv.P.nnz),
            'smoother_kind': lv.f_smoother.kind,
            'smoother_order': int(lv.f_smoother.order),
            'smoother_effective_order': int(lv.f_smoother.effective_order),
            'nnz_smoother_assembled': None if lv.f_smoother_assembled is None
            else int(lv.f_smoother_assembled.nnz),
        })
    return {
        'num_levels': len(H.levels), 'num_grids': len(H.levels) + 1,
        'n_top': int(H.top_A.nrows), 'nnz_top': int(H.top_A.nnz), 'levels': levels,
        'coarsest': {
            'n': int(H.coarsest_A.nrows), 'nnz': int(H.coarsest_A.nnz),
            'solver_kind': H.coarse_solver.kind, 'solver_order': int(H.coarse_solver.order),
            'solver_effective_order': int(H.coarse_solver.effective_order),
        },
        'truncated_at': H.truncated_at,
        'cycle_complexity': H.cycle_complexity,
        'storage_complexity': H.storage_complexity,
        'grid_complexity': H.grid_complexity,
    }


class _Timer:
    """Per-phase time accumulation (hierarchy.py:184-197).  CUDA events are
    recorded on the setup stream at both ends of the phase (in stream order,
    so the phase owns its kernels and any device idle time inside it); the
    elapsed times are summed by _flush_timings once at the end of the level
    loop, instead of synchronising the device twice per phase."""

    def __init__(self, sink, phase):
        self.sink = sink
        self.phase = phase

    def _stream(self):
        # the setup stream, looked up once per setup (torch's current_stream()
        # costs ~10 us of device-index bookkeeping per record)
        import torch
        st = self.sink.get('_stream')
        if st is None:
            st = self.sink['_stream'] = torch.cuda.current_stream()
        return st

    def __enter__(self):
        import torch
        if self.sink is not None:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e0.record(self._stream())
        return self

    def __exit__(self, *exc):
        import torch
        if self.sink is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(self._stream())
            self.sink.setdefault('_pending', []).append((self.phase, self.sink.get('_level'),
                                                         self.e0, e1))
        return False


def _flush_timings(sink):
    """Sum the recorded phase events into seconds (one synchronisation);
    per-level sums go to sink['_per_level'][level][phase]."""
    pend = sink.pop('_pending', None) if sink is not None else None
    if not pend:
        return
    pend[-1][3].synchronize()
    per = sink.setdefault('_per_level', {})
    for phase, level, e0, e1 in pend:
        dt = e0.elapsed_time(e1) / 1e3
        sink[phase] = sink.get(phase, 0.0) + dt
        if level is not None:
            d = per.setdefault(level, {})
            d[phase] = d.get(phase, 0.0) + dt


def resolve_truncate_start(cfg, n_top):
    """A-priori truncation start level (hierarchy.py:318-333)."""
    if cfg.auto_truncate_start_level is not None:
        return cfg.auto_truncate_start_level
    reach = cfg.coarsest_poly_order + 1
    if n_top <= reach:
        return 0
    return int(np.ceil(np.log2(n_top / reach))) + 2


# ---------------------------------------------------------------------------
# level operators
# ---------------------------------------------------------------------------

def _colmaps(split):
    """Device column maps old -> F position / C position (-1 elsewhere)."""
    from . import _lib as L
    from .csr import IDX, empty
    n = split.n
    fmap, cmap = empty(n, IDX), empty(n, IDX)
    L.call('airg_label_colmap', n, L.ptr(split.labels), 0, L.ptr(split.pos), L.ptr(fmap),
           L.stream_handle())
    L.call('airg_label_colmap', n, L.ptr(split.labels), 1, L.ptr(split.pos), L.ptr(cmap),
           L.stream_handle())
    return fmap, cmap


def _smoother_for(A_ff, cfg, seed):
    from .gmres_poly import gmres_poly_arnoldi, neumann_poly
    if cfg.inverse_type == 'arnoldi':
        return gmres_poly_arnoldi(A_ff, cfg.poly_order, seed)
    return neumann_poly(A_ff, cfg.poly_order)


def build_restriction(A, split, cfg, level=0, timings=None, return_assembled=False,
                      smoother=None):
    """R = [Z I] with Z = -A_cf Ahat_ff, Ahat the fixed-sparsity polynomial
    (hierarchy.py:211-247).  ``smoother`` injects a precomputed polynomial."""
    import ctypes as C
    from . import _lib as L
    from .csr import drop_and_lump, extract_mapped, spgemm, take
    from .gmres_poly import assemble_fixed_sparsity
    with _Timer(timings, 'extract'):
        fmap, cmap = _colmaps(split)
        A_ff = extract_mapped(A, split.f_idx, fmap, split.n_f)
        A_fc = extract_mapped(A, split.f_idx, cmap, split.n_c)
        A_cf = extract_mapped(A, split.c_idx, fmap, split.n_f)
    with _Timer(timings, 'polynomial'):
        if smoother is None:
            smoother = _smoother_for(A_ff, cfg, derive_seed(cfg.seed, level, SEED_SMOOTHER))
        assembled = assemble_fixed_sparsity(smoother, A_ff)
    with _Timer(timings, 'spgemm_R'):
        Z = spgemm(A_cf, assembled, negate=True)
    with _Timer(timings, 'drop'):
        Z = drop_and_lump(Z, cfg.r_drop, lump=False)
    with _Timer(timings, 'spgemm_R'):
        r = C.c_void_p()
        L.call('airg_restriction', A.nrows, split.n_c, L.ptr(Z.row_offsets),
               L.ptr(Z.col_indices), L.ptr(Z.values), L.ptr(split.f_idx), L.ptr(split.c_idx),
               C.byref(r), L.stream_handle())
        R = take(r)
    if return_assembled:
        return R, A_ff, A_fc, smoother, assembled
    return R, A_ff, A_fc, smoother


def _prolong_cols(A, split):
    from . import _lib as L
    from .csr import IDX, empty
    pcol = empty(split.n, IDX)
    L.call('airg_prolong_onepoint', split.n, L.ptr(A.row_offsets), L.ptr(A.col_indices),
           L.ptr(A.values), L.ptr(split.labels), L.ptr(split.pos), L.ptr(pcol), L.stream_handle())
    return pcol


def build_prolongation(A, split, pcol=None):
    """One-point classical prolongator P = [W; I] (hierarchy.py:250-278)."""
    import torch
    from .csr import IDX, VAL, SparseMatrix
    n = split.n
    if split.n_f == 0:
        return SparseMatrix.identity(n)
    if pcol is None:
        pcol = _prolong_cols(A, split)
    dev = pcol.device
    return SparseMatrix(n, split.n_c, torch.arange(n + 1, dtype=IDX, device=dev), pcol,
                        torch.ones(n, dtype=VAL, device=dev))


def coarse_matrix(A, R, P, cfg, timings=None):
    """drop_and_lump(R (A P), a_drop, lump) with the drop fused into the
    numeric SpGEMM epilogue (hierarchy.py:281-286)."""
    import ctypes as C
    from . import _lib as L
    from .csr import spgemm, take
    with _Timer(timings, 'spgemm_coarse'):
        if P.nnz == P.nrows and A.nrows == P.nrows:
            r = C.c_void_p()
            L.call('airg_galerkin', A.nrows, R.nrows, L.ptr(R.row_offsets), L.ptr(R.col_indices),
                   L.ptr(R.values), L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
                   L.ptr(P.col_indices), float(cfg.a_drop), 1 if cfg.lump else 0, C.byref(r),
                   L.stream_handle())
            return take(r)
        from .csr import drop_and_lump
        return drop_and_lump(spgemm(R, spgemm(A, P)), cfg.a_drop, cfg.lump)


def _repair_split(A, split):
    """F points without a C coupling become C (hierarchy.py:289-305)."""
    import ctypes as C
    from . import _lib as L
    from .cfsplit import CFSplit
    if split.n_f == 0:
        return split
    lab = split.labels.clone()
    ch = C.c_int32()
    L.call('airg_repair_split', split.n, L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(lab),
           C.byref(ch), L.stream_handle())
    if ch.value == 0:
        return split
    return CFSplit.from_labels(lab)


def _build_coarse_solver(A, cfg, level):
    from .gmres_poly import gmres_poly_arnoldi, gmres_poly_newton, neumann_poly
    seed = derive_seed(cfg.seed, level, SEED_COARSE_POLY)
    kind = cfg.coarsest_inverse_type
    if kind == 'newton':
        return gmres_poly_newton(A, cfg.coarsest_poly_order, seed)
    if kind == 'arnoldi':
        return gmres_poly_arnoldi(A, cfg.coarsest_poly_order, seed)
    return neumann_poly(A, cfg.coarsest_poly_order)


def try_truncate(A, cfg, level, start_level=None, solver=None):
    """Tentative high-order coarse solver test (hierarchy.py:336-362)."""
    from .csr import norm2, random_unit_vector, spmv
    from .gmres_poly import apply_matrix_free
    if start_level is None:
        start_level = resolve_truncate_start(cfg, A.nrows)
    if cfg.auto_truncate_tol is None or level < start_level:
        return None
    if solver is None:
        try:
            solver = _build_coarse_solver(A, cfg, level)
        except (ValueError, np.linalg.LinAlgError) as exc:
            _log.warning('tentative coarse solver failed at level %d: %s', level, exc)
            return None
    rhs = random_unit_vector(A.nrows, derive_seed(cfg.seed, level, SEED_TRUNC_RHS))
    x = apply_matrix_free(solver, A, rhs)
    residual = norm2(rhs - spmv(A, x)) / norm2(rhs)
    if np.isfinite(residual) and residual <= cfg.auto_truncate_tol:
        return solver
    return None


def setup(A, cfg, poly_inject=None, keep_level_matrices=False):
    """Build the multigrid hierarchy on the GPU (hierarchy.py:365-448).

    ``poly_inject`` (test hook, not in the reference API): dict mapping
    ('smoother', level) / ('coarse', level) to PolySolver objects used instead
    of recomputing them -- coefficient injection, SURVEY.md 8(c).
    The recorded polynomials of a run are in ``H.polys``.
    """
    from .cfsplit import cf_split
    from .csr import as_matrix
    cfg.validate()
    A = as_matrix(A)  # a reference airmg.SparseMatrix (host, int64) is uploaded
    if A.nrows != A.ncols:
        raise ValueError('require a square matrix')
    if A.nrows == 0:
        raise ValueError('require a non-empty matrix')
    inj = poly_inject or {}
    polys = {}
    timings = {phase: 0.0 for phase in SETUP_PHASES}
    truncate_start = resolve_truncate_start(cfg, A.nrows)
    levels, current, coarse_solver, truncated_at = build_levels(
        A, cfg, 0, truncate_start, inj, polys, timings, keep_level_matrices)
    per_level = timings.pop('_per_level', {})
    H = Hierarchy(levels=levels, coarsest_A=current, coarse_solver=coarse_solver, top_A=A,
                  truncated_at=truncated_at, config=cfg, setup_breakdown=timings)
    H.setup_levels = per_level  # {level: {phase: seconds}}
    H.polys = polys
    return finalize_complexities(H)


def build_levels(A, cfg, level0, truncate_start, inj, polys, timings, keep_level_matrices=False):
    """The level loop of setup (hierarchy.py:386-434) from level index
    ``level0`` on a (replicated) level matrix ``A``.  Returns (levels,
    coarsest matrix, coarse solver, truncated_at)."""
    from .cfsplit import cf_split
    levels = []
    current = A
    level = level0
    truncated_at = None
    coarse_solver = None

    def coarse_here(M, lev):
        with _Timer(timings, 'truncation'):
            s = inj.get(('coarse', lev)) or _build_coarse_solver(M, cfg, lev)
        polys[('coarse', lev)] = s
        return s

    while True:
        timings['_level'] = level
        if current.nrows <= cfg.min_coarse_size:
            coarse_solver = coarse_here(current, level)
            break
        if level >= cfg.max_levels:
            _log.warning('level budget (%d) exhausted at %d unknowns; building the coarse '
                         'solver here', cfg.max_levels, current.nrows)
            coarse_solver = coarse_here(current, level)
            break
        with _Timer(timings, 'truncation'):
            cand = None
            if cfg.auto_truncate_tol is not None and level >= truncate_start:
                cand = try_truncate(current, cfg, level, start_level=truncate_start,
                                    solver=inj.get(('coarse', level)))
        if cand is not None:
            coarse_solver = cand
            polys[('coarse', level)] = cand
            truncated_at = level
            break
        with _Timer(timings, 'cf_split'):
            split, ddc_stats = cf_split(current, cfg.strong_threshold, cfg.ddc_fraction,
                                        cfg.ddc_its, derive_seed(cfg.seed, level, SEED_SPLIT),
                                        nbins=cfg.ddc_bins)
        if split.n_c == split.n:
            raise ValueError(f'splitting produced no F points at level {level}')
        if split.n_c > 0:
            with _Timer(timings, 'cf_split'):
                split = _repair_split(current, split)
        if split.n_c == 0 or split.n_f == 0:
            _log.info('level %d needs no further reduction; building the coarse solver '
                      'directly', level)
            coarse_solver = coarse_here(current, level)
            break
        R, A_ff, A_fc, smoother, assembled = build_restriction(
            current, split, cfg, level=level, timings=timings, return_assembled=True,
            smoother=inj.get(('smoother', level)))
        polys[('smoother', level)] = smoother
        with _Timer(timings, 'prolongator'):
            P = build_prolongation(current, split)
        coarse = coarse_matrix(current, R, P, cfg, timings=timings)
        levels.append(Level(R=R, P=P, A_ff=A_ff, A_fc=A_fc, f_smoother=smoother, split=split,
                            n=current.nrows, nnz_A=current.nnz,
                            f_smoother_assembled=None if cfg.matrix_free_polys else assembled,
                            ddc_stats=tuple(ddc_stats)))
        if keep_level_matrices:
            levels[-1].A = current
        current = coarse
        level += 1
    _flush_timings(timings)
    timings.pop('_level', None)
    timings.pop('_stream', None)
    return levels, current, coarse_solver, truncated_at
