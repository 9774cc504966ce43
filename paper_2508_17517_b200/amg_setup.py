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
    """Per-phase wall-clock accumulation (hierarchy.py:184-197); the device
    is synchronised at both ends so the phase owns its kernels."""

    def __init__(self, sink, phase):
        self.sink = sink
        self.phase = phase

    def __enter__(self):
        import torch
        torch.cuda.synchronize()
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        import torch
        torch.cuda.synchronize()
        if self.sink is not None:
            self.sink[self.phase] = self.sink.get(self.phase, 0.0) + time.perf_counter() - self.t0
        return False


def resolve_truncate_start(cfg, n_top):
    """A-priori truncation start level (hierarchy.py:318-333)."""
    if cfg.auto_truncate_start_level is not None:
        return cfg.auto_truncate_start_level
    reach = cfg.coarsest_poly_order + 1
    if n_top <= reach:
        return 0
    return int(np.ceil(np.log2(n_top / reach))) + 2
