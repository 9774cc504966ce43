"""Generate the golden fixtures from the REAL reference package (airmg).

Run in the build container (the only place /root/reference exists):

    OPENBLAS_NUM_THREADS=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Outputs ``tests/golden/*.npz``.  The fixtures pin the oracle
(``oracle/airg_oracle.py``); ``tests/test_oracle_golden.py`` checks them.
Large arrays are stored as sha256 digests of their raw bytes (int64 indices,
float64 values) so the fixtures stay small while still pinning every bit.
"""

import hashlib
import os
import sys

import numpy as np

os.environ.setdefault('OPENBLAS_NUM_THREADS', '1')
sys.path.insert(0, '/root/reference/pkg/src')
import airmg  # noqa: E402
import airmg.hierarchy as hmod  # noqa: E402
from airmg.polynomial import _random_unit_vector  # noqa: E402
from airmg.splitting import _luby_ranks  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
PI4 = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_digest(M):
    return digest(np.asarray(M.row_offsets, np.int64), np.asarray(M.col_indices, np.int64),
                  np.asarray(M.values, np.float64))


def capture_setup(A, cfg):
    """Run the reference setup, recording each level matrix handed to cf_split."""
    mats = []
    orig = hmod.cf_split

    def spy(M, *a, **k):
        mats.append(M)
        return orig(M, *a, **k)

    hmod.cf_split = spy
    try:
        H = airmg.setup(A, cfg)
    finally:
        hmod.cf_split = orig
    return H, mats


def hierarchy_case(name, nx, ny, v, cfg, full):
    A, b = airmg.build_advection_2d(airmg.AdvectionProblem(nx=nx, ny=ny, vx=v[0], vy=v[1]))
    H, mats = capture_setup(A, cfg)
    x, st = airmg.richardson_solve(H, b, np.ones(A.nrows), airmg.SolveConfig())
    out = dict(nx=nx, ny=ny, vx=v[0], vy=v[1], nlev=len(H.levels),
               truncated_at=-1 if H.truncated_at is None else H.truncated_at,
               history=np.array(st.residual_history), iterations=st.iterations,
               x_digest=digest(x), x_head=x[:64].copy(),
               cycle_complexity=H.cycle_complexity,
               storage_complexity=H.storage_complexity,
               grid_complexity=H.grid_complexity,
               flops=airmg.count_cycle_flops(H),
               coarse_roots=H.coarse_solver.roots if H.coarse_solver.roots is not None
               else np.zeros(0, np.complex128),
               coarse_eff=H.coarse_solver.effective_order,
               coarsest_digest=csr_digest(H.coarsest_A), coarsest_n=H.coarsest_A.nrows,
               coarsest_nnz=H.coarsest_A.nnz)
    cfg_d = cfg.to_dict()
    for k, val in cfg_d.items():
        out['cfg_' + k] = -1 if val is None else val
    for i, L in enumerate(H.levels):
        p = f'L{i}_'
        out[p + 'labels'] = L.split.labels
        out[p + 'coeffs'] = L.f_smoother.coeffs
        out[p + 'eff'] = L.f_smoother.effective_order
        out[p + 'ddc'] = np.array([[s.n_f_before, s.converted, s.ratio_min, s.ratio_max,
                                    s.cut] for s in L.ddc_stats], dtype=np.float64)
        for nm, M in (('R', L.R), ('P', L.P), ('Aff', L.A_ff), ('Afc', L.A_fc),
                      ('A', mats[i])):
            out[p + nm + '_digest'] = csr_digest(M)
            out[p + nm + '_nnz'] = M.nnz
            if full:
                out[p + nm + '_ptr'] = M.row_offsets
                out[p + nm + '_col'] = M.col_indices
                out[p + nm + '_val'] = M.values
    if full:
        C = H.coarsest_A
        out['C_ptr'], out['C_col'], out['C_val'] = C.row_offsets, C.col_indices, C.values
    np.savez_compressed(os.path.join(OUT, name + '.npz'), **out)
    print(name, 'levels', len(H.levels), 'its', st.iterations, 'hist', st.residual_history[-1])


def kernels_case():
    """Small KATs for the individual kernels and the random streams."""
    rng = np.random.default_rng(1234)
    out = {}
    # PCG64 streams (splitting.py:119, polynomial.py:63) and seed derivation
    for s in (0, 7, 123456789):
        out[f'pcg_random_{s}'] = np.random.default_rng(np.random.SeedSequence(s)).random(257)
        out[f'unit_{s}'] = _random_unit_vector(257, s)
    out['derived_seeds'] = np.array([[r, l, role, hmod._derive_seed(r, l, role)]
                                     for r in (0, 5) for l in range(20) for role in range(4)],
                                    dtype=np.int64)
    deg = rng.integers(0, 9, 500).astype(np.float64)
    out['luby_deg'] = deg
    out['luby_ranks'] = _luby_ranks(500, deg, 99)
    # random CSR operands with cancellations
    def rnd(m, n, dens, seed):
        r = np.random.default_rng(seed)
        d = r.standard_normal((m, n)) * (r.random((m, n)) < dens)
        return airmg.SparseMatrix.from_dense(np.round(d, 1))
    A = rnd(60, 50, 0.15, 1)
    B = rnd(50, 70, 0.15, 2)
    Pm = rnd(60, 70, 0.3, 3)
    for nm, M in (('A', A), ('B', B), ('Pm', Pm)):
        out[nm + '_ptr'], out[nm + '_col'], out[nm + '_val'] = M.row_offsets, M.col_indices, M.values
    for nm, M in (('AB', airmg.spgemm(A, B)), ('ABmask', airmg.spgemm_fixed_sparsity(A, B, Pm))):
        out[nm + '_ptr'], out[nm + '_col'], out[nm + '_val'] = M.row_offsets, M.col_indices, M.values
    S = rnd(80, 80, 0.1, 4)
    S = airmg.SparseMatrix.from_dense(S.to_dense() + np.diag(np.linspace(1, 3, 80)))
    out['S_ptr'], out['S_col'], out['S_val'] = S.row_offsets, S.col_indices, S.values
    D = airmg.drop_and_lump(S, 0.5, True)
    out['Sdrop_ptr'], out['Sdrop_col'], out['Sdrop_val'] = D.row_offsets, D.col_indices, D.values
    g = airmg.strength_graph(S, 0.5)
    out['Sclo_ptr'], out['Sclo_col'] = g.symmetric_closure.row_offsets, g.symmetric_closure.col_indices
    split, stats = airmg.cf_split(S, 0.5, 0.1, 2, 11)
    out['S_labels'] = split.labels
    out['S_ddc'] = np.array([[s.n_f_before, s.converted, s.ratio_min, s.ratio_max, s.cut]
                             for s in stats])
    p = airmg.gmres_poly_arnoldi(S, 4, 5)
    out['S_coeffs'] = p.coeffs
    Ah = airmg.assemble_fixed_sparsity(p, S)
    out['Shat_ptr'], out['Shat_col'], out['Shat_val'] = Ah.row_offsets, Ah.col_indices, Ah.values
    pn = airmg.gmres_poly_newton(S, 30, 5)
    out['S_roots'] = pn.roots
    bvec = rng.standard_normal(80)
    out['bvec'] = bvec
    out['S_newton_apply'] = airmg.apply_matrix_free(pn, S, bvec)
    out['S_horner_apply'] = airmg.apply_matrix_free(p, S, bvec)
    np.savez_compressed(os.path.join(OUT, 'kernels.npz'), **out)
    print('kernels ok')


if __name__ == '__main__':
    kernels_case()
    hierarchy_case('adv32_o4', 32, 32, PI4, airmg.SetupConfig(poly_order=4), full=True)
    hierarchy_case('adv48x40_hard_o6', 48, 40, (float(np.sqrt(2 / 3)), float(np.sqrt(1 / 3))),
                   airmg.SetupConfig(strong_threshold=0.4), full=True)
    hierarchy_case('adv128_o4', 128, 128, PI4, airmg.SetupConfig(poly_order=4), full=False)
    hierarchy_case('adv128_o6', 128, 128, PI4, airmg.SetupConfig(), full=False)
    hierarchy_case('adv64_trunc4', 64, 64, PI4,
                   airmg.SetupConfig(poly_order=4, auto_truncate_start_level=3), full=False)
