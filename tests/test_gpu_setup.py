"""GPU parity of the setup path against the oracle and the reference's own
golden fixtures.  Everything here is BITWISE (integer / pattern work and
the sequential-sum fp64 kernels), except the Krylov coefficients, which
use device dot products (<= 1e-12 relative) and are therefore injected
when whole hierarchies are compared."""

import hashlib

import numpy as np
import pytest

from oracle import airg_oracle as O
from tests.gpu_util import dev_csr, dev_poly, host_csr, oracle_poly, rel, upload_hierarchy, tonp

pytestmark = pytest.mark.gpu

PI4 = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
HARD = (float(np.sqrt(2 / 3)), float(np.sqrt(1 / 3)))


@pytest.fixture(scope='module')
def G():
    import paper_2508_17517_b200 as G
    return G


def same(M_dev, M_or):
    H = host_csr(M_dev)
    assert (H.nrows, H.ncols) == (M_or.nrows, M_or.ncols)
    assert np.array_equal(H.ptr, M_or.ptr)
    assert np.array_equal(H.col, M_or.col)
    assert H.val.tobytes() == M_or.val.tobytes()


def digest(M):
    H = host_csr(M)
    h = hashlib.sha256()
    for a in (H.ptr.astype(np.int64), H.col.astype(np.int64), H.val.astype(np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope='module')
def hier():
    A = O.advection_2d(64, 64, *PI4)
    return O.setup(A, O.Cfg(poly_order=4), keep_level_matrices=True)


@pytest.fixture(scope='module')
def hier_hard():
    A = O.advection_2d(48, 40, *HARD)
    return O.setup(A, O.Cfg(strong_threshold=0.4), keep_level_matrices=True)


def level_mats(h):
    return [L.A for L in h.levels] + [h.coarsest_A]


def test_generator_bitwise(G):
    for nx, ny, v in [(64, 64, PI4), (37, 5, HARD), (1, 9, PI4), (9, 1, PI4), (5, 4, (1.0, 0.0)),
                      (5, 4, (0.0, 2.0))]:
        A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=ny, vx=v[0], vy=v[1]))
        same(A, O.advection_2d(nx, ny, *v))
        assert float(b.abs().max()) == 0.0 if b.numel() else True
    same(G.build_advection_1d(17, 1.5), O.advection_1d(17, 1.5))


def test_pcg64_stream_bitwise(G, golden):
    from paper_2508_17517_b200.csr import pcg_vector, random_unit_vector
    g = golden('kernels')
    for s in (0, 7, 123456789):
        assert pcg_vector(s, 257, 0.0, 1.0).cpu().numpy().tobytes() == g[f'pcg_random_{s}'].tobytes()
        raw = np.random.default_rng(np.random.SeedSequence(s)).uniform(-1.0, 1.0, 100003)
        assert pcg_vector(s, 100003, -1.0, 2.0).cpu().numpy().tobytes() == raw.tobytes()
        u = random_unit_vector(257, s).cpu().numpy()
        assert rel(u, g[f'unit_{s}']) < 1e-14


def test_strength_graph_bitwise(G, hier, hier_hard):
    for h, theta in ((hier, 0.99), (hier_hard, 0.4), (hier, 0.0), (hier, 0.5)):
        for M in level_mats(h):
            S_o, C_o = O.strength(M, theta)
            g = G.strength_graph(dev_csr(M), theta)
            same(g.S, S_o)
            same(g.symmetric_closure, C_o)


def test_cf_split_bitwise(G, hier, hier_hard):
    for h, theta in ((hier, 0.99), (hier_hard, 0.4)):
        for lev, M in enumerate(level_mats(h)):
            for its, seed in ((2, 1 + lev), (3, 17)):
                lab_o, st_o = O.cf_split(M, theta, 0.01, its, seed)
                split, st = G.cf_split(dev_csr(M), theta, 0.01, its, seed)
                assert np.array_equal(split.labels_host(), lab_o), lev
                assert len(st) == len(st_o)
                for a, b in zip(st, st_o):
                    assert (a.n_f_before, a.converted) == (b['n_f_before'], b['converted'])
                    assert (a.ratio_min, a.ratio_max, a.cut) == (b['ratio_min'], b['ratio_max'],
                                                                 b['cut'])
                    assert abs(a.ratio_mean - b['ratio_mean']) <= 1e-12 * abs(b['ratio_mean'])


def test_pmisr_loop_cap_and_kats(G, golden):
    g = golden('kernels')
    S = O._mk(80, 80, g['S_ptr'], g['S_col'], g['S_val'])
    split, stats = G.cf_split(dev_csr(S), 0.5, 0.1, 2, 11)
    assert np.array_equal(split.labels_host(), g['S_labels'])
    _, clo = O.strength(O.advection_2d(40, 40, *PI4), 0.99)
    for cap in (0, 1, 2, None):
        lab_o, _ = O.pmisr_labels(clo, 5, cap)
        graph = G.StrengthGraph(dev_csr(clo), dev_csr(clo))
        assert np.array_equal(G.pmisr(graph, 5, max_luby_loops=cap).labels_host(), lab_o)


def test_ddc_errors_and_kat(G):
    # zero diagonal in the fine block
    A = O.from_triplets(3, 3, [0, 1, 1, 2], [0, 0, 1, 1], [1.0, -1.0, 0.0, 2.0])
    lab = G.CFSplit.from_labels(np.array([0, 0, 1], np.int8))
    with pytest.raises(ValueError, match='zero diagonal'):
        G.ddc_pass(dev_csr(A), lab, 0.1)
    # binning rule (tests/test_splitting.py:167-179 style): ratios {0.1, 0.5, 0.9, 1.3}
    n = 4
    rows, cols, vals = [], [], []
    for i, r in enumerate([0.1, 0.5, 0.9, 1.3]):
        rows += [i, i]
        cols += [i, (i + 1) % n]
        vals += [1.0, r]
    A = O.from_triplets(n, n, rows, cols, vals)
    lab = np.zeros(n, np.int8)
    want, st_o = O.ddc(A, lab, 0.25, 1000)
    from paper_2508_17517_b200.cfsplit import _ddc_core
    got, st = _ddc_core(dev_csr(A), G.CFSplit.from_labels(lab), 0.25, 1000)
    assert np.array_equal(got.labels_host(), want)
    assert st.cut == st_o['cut']


def test_extract_spgemm_masked_drop_bitwise(G, golden, hier):
    g = golden('kernels')
    A = O._mk(60, 50, g['A_ptr'], g['A_col'], g['A_val'])
    B = O._mk(50, 70, g['B_ptr'], g['B_col'], g['B_val'])
    Pm = O._mk(60, 70, g['Pm_ptr'], g['Pm_col'], g['Pm_val'])
    same(G.spgemm(dev_csr(A), dev_csr(B)), O.spgemm(A, B))
    same(G.spgemm_fixed_sparsity(dev_csr(A), dev_csr(B), dev_csr(Pm)), O.spgemm_masked(A, B, Pm))
    S = O._mk(80, 80, g['S_ptr'], g['S_col'], g['S_val'])
    same(G.drop_and_lump(dev_csr(S), 0.5, True), O.drop_lump(S, 0.5, True))
    same(G.drop_and_lump(dev_csr(S), 0.5, False), O.drop_lump(S, 0.5, False))
    rng = np.random.default_rng(5)
    for L in hier.levels:
        M = L.A
        rows = np.sort(rng.choice(M.nrows, M.nrows // 2, replace=False))
        cols = np.sort(rng.choice(M.ncols, M.ncols // 3, replace=False))
        same(G.extract(dev_csr(M), rows, cols), O.submatrix(M, rows, cols))
        same(G.spgemm(dev_csr(L.R), dev_csr(M)), O.spgemm(L.R, M))
        same(G.spgemm(dev_csr(M), dev_csr(L.P)), O.spgemm(M, L.P))
        same(G.drop_and_lump(dev_csr(O.spgemm(M, M)), 1e-3, True),
             O.drop_lump(O.spgemm(M, M), 1e-3, True))


def test_empty_and_ragged_products(G):
    E = O.from_triplets(4, 3, [], [], [])
    B = O.from_triplets(3, 5, [0, 2], [4, 1], [1.0, -2.0])
    same(G.spgemm(dev_csr(E), dev_csr(B)), O.spgemm(E, B))
    A = O.from_triplets(4, 3, [1, 1, 3], [0, 2, 2], [2.0, 1.0, -1.0])
    same(G.spgemm(dev_csr(A), dev_csr(B)), O.spgemm(A, B))
    # exact cancellation kept as a structural zero
    A = O.from_triplets(1, 2, [0, 0], [0, 1], [1.0, 1.0])
    B = O.from_triplets(2, 1, [0, 1], [0, 0], [1.0, -1.0])
    C = G.spgemm(dev_csr(A), dev_csr(B))
    assert C.nnz == 1 and float(C.values[0]) == 0.0
    with pytest.raises(ValueError):
        G.spgemm(dev_csr(B), dev_csr(B))


def test_long_rows_use_fallback_paths(G):
    """Rows beyond the shared-memory classes (global-table fallbacks)."""
    rng = np.random.default_rng(7)
    n = 6000
    r = np.repeat(np.arange(3), 2500)
    c = np.concatenate([rng.choice(n, 2500, replace=False) for _ in range(3)])
    A = O.from_triplets(3, n, r, c, rng.standard_normal(len(r)))
    B = O.from_triplets(n, n, np.arange(n), (np.arange(n) * 7) % n, rng.standard_normal(n))
    B2 = O.from_triplets(n, n, np.concatenate([np.arange(n), np.arange(n)]),
                         np.concatenate([(np.arange(n) * 7) % n, (np.arange(n) * 11 + 1) % n]),
                         rng.standard_normal(2 * n))
    same(G.spgemm(dev_csr(A), dev_csr(B)), O.spgemm(A, B))
    same(G.spgemm(dev_csr(A), dev_csr(B2)), O.spgemm(A, B2))


def test_poly_assembly_bitwise(G, golden, hier, hier_hard):
    g = golden('kernels')
    S = O._mk(80, 80, g['S_ptr'], g['S_col'], g['S_val'])
    p = O.Poly('arnoldi_coeff', 4, 4, coeffs=g['S_coeffs'])
    same(G.assemble_fixed_sparsity(dev_poly(p), dev_csr(S)), O.assemble_poly(p, S))
    for h in (hier, hier_hard):
        for L in h.levels:
            same(G.assemble_fixed_sparsity(dev_poly(L.smoother), dev_csr(L.A_ff)),
                 O.assemble_poly(L.smoother, L.A_ff))
    # degree 0 keeps the full diagonal even for c0 = 0
    p0 = O.Poly('arnoldi_coeff', 0, 0, coeffs=np.array([0.0]))
    same(G.assemble_fixed_sparsity(dev_poly(p0), dev_csr(S)), O.assemble_poly(p0, S))


def test_level_operators_bitwise(G, hier, hier_hard):
    for h, cfg in ((hier, O.Cfg(poly_order=4)), (hier_hard, O.Cfg(strong_threshold=0.4))):
        gcfg = G.SetupConfig(**{k: getattr(cfg, k) for k in O.Cfg.__dataclass_fields__})
        for lev, L in enumerate(h.levels):
            A = dev_csr(L.A)
            split = G.CFSplit.from_labels(L.labels)
            R, A_ff, A_fc, sm = G.build_restriction(A, split, gcfg, level=lev,
                                                    smoother=dev_poly(L.smoother))
            same(R, L.R)
            same(A_ff, L.A_ff)
            same(A_fc, L.A_fc)
            P = G.build_prolongation(A, split)
            same(P, L.P)
            nxt = G.coarse_matrix(A, R, P, gcfg)
            want = h.levels[lev + 1].A if lev + 1 < len(h.levels) else h.coarsest_A
            same(nxt, want)


def test_krylov_coefficients_close_to_oracle(G, hier):
    for lev, L in enumerate(hier.levels):
        seed = O.derive_seed(0, lev, O.ROLE_SMOOTHER)
        p = G.gmres_poly_arnoldi(dev_csr(L.A_ff), 4, seed)
        assert p.effective_order == L.smoother.effective_order
        assert np.max(np.abs(p.coeffs - L.smoother.coeffs)) <= 1e-10 * np.max(np.abs(L.smoother.coeffs))
    C = hier.coarsest_A
    pn = G.gmres_poly_newton(dev_csr(C), 100, O.derive_seed(0, len(hier.levels), O.ROLE_COARSE))
    assert pn.effective_order == hier.coarse_solver.effective_order
    # root clusters near sqrt(2) make the stability-copy count (1e-4 relative gap,
    # polynomial.py:238-254) rounding-sensitive; both polynomials must solve C
    assert abs(len(pn.roots) - len(hier.coarse_solver.roots)) <= 4
    b = np.random.default_rng(0).standard_normal(C.nrows)
    x = G.apply_matrix_free(pn, dev_csr(C), b).cpu().numpy()
    assert np.linalg.norm(b - O.spmv(C, x)) <= 1e-8 * np.linalg.norm(b)


def _inject_from_fixture(G, g):
    inj = {}
    for i in range(int(g['nlev'])):
        inj[('smoother', i)] = G.PolySolver('arnoldi_coeff', int(g['cfg_poly_order']),
                                            int(g[f'L{i}_eff']), coeffs=g[f'L{i}_coeffs'])
    lev = int(g['nlev'])
    inj[('coarse', lev)] = G.PolySolver('newton_roots', int(g['cfg_coarsest_poly_order']),
                                        int(g['coarse_eff']), roots=g['coarse_roots'])
    return inj


def _cfg(G, g):
    kw = {}
    for f in O.Cfg.__dataclass_fields__:
        v = g['cfg_' + f].item()
        if f == 'auto_truncate_start_level' and v == -1:
            v = None
        kw[f] = v
    return G.SetupConfig(**kw)


@pytest.mark.parametrize('case', ['adv32_o4', 'adv48x40_hard_o6', 'adv128_o4', 'adv128_o6',
                                  'adv64_trunc4'])
def test_setup_matches_reference_fixtures(G, golden, case):
    """Inject the REFERENCE's coefficients/roots into the GPU setup: every
    level's labels and R / P / A_ff / A_fc / A digests must equal the ones the
    reference package produced (tests/golden/make_golden.py)."""
    g = golden(case)
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=int(g['nx']), ny=int(g['ny']),
                                                   vx=float(g['vx']), vy=float(g['vy'])))
    H = G.setup(A, _cfg(G, g), poly_inject=_inject_from_fixture(G, g), keep_level_matrices=True)
    assert H.num_levels == int(g['nlev'])
    assert (H.truncated_at if H.truncated_at is not None else -1) == int(g['truncated_at'])
    for i, L in enumerate(H.levels):
        p = f'L{i}_'
        assert np.array_equal(L.split.labels_host(), g[p + 'labels']), i
        for nm, M in (('R', L.R), ('P', L.P), ('Aff', L.A_ff), ('Afc', L.A_fc), ('A', L.A)):
            assert digest(M) == str(g[p + nm + '_digest']), (i, nm)
    assert digest(H.coarsest_A) == str(g['coarsest_digest'])
    assert H.cycle_complexity == pytest.approx(float(g['cycle_complexity']), rel=1e-14)
    # parity mode: reference arithmetic order in every kernel -> x is the
    # reference's bit for bit; only the norm reduction order differs.
    x, st = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig(), exact=True)
    assert st.iterations == int(g['iterations'])
    h = hashlib.sha256(np.ascontiguousarray(tonp(x)).tobytes()).hexdigest()
    assert h == str(g['x_digest'])
    assert rel(st.residual_history, g['history']) < 1e-13
    # fast mode (vector SpMV + FMA): same iterations, history within 1e-10 of
    # the initial residual
    x, st = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig())
    assert st.iterations == int(g['iterations'])
    assert np.max(np.abs(np.array(st.residual_history) - g['history'])) <= 1e-10 * g['history'][0]


@pytest.mark.parametrize('nx,ny,v,order', [(64, 64, PI4, 4), (128, 128, PI4, 6),
                                           (48, 40, HARD, 6), (256, 256, PI4, 4)])
def test_gpu_setup_replayed_by_oracle(G, nx, ny, v, order):
    """GPU setup with its own device Krylov coefficients; the oracle replays
    it with those coefficients injected: hierarchies identical, histories
    within 1e-10."""
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=ny, vx=v[0], vy=v[1]))
    cfg = G.SetupConfig(poly_order=order)
    H = G.setup(A, cfg, keep_level_matrices=True)
    inj = {k: oracle_poly(p) for k, p in H.polys.items()}
    Ao = O.advection_2d(nx, ny, *v)
    Ho = O.setup(Ao, O.Cfg(poly_order=order), poly_inject=inj, keep_level_matrices=True)
    assert H.num_levels == len(Ho.levels)
    assert H.truncated_at == Ho.truncated_at
    for L, Lo in zip(H.levels, Ho.levels):
        assert np.array_equal(L.split.labels_host(), Lo.labels)
        for a, o in ((L.R, Lo.R), (L.P, Lo.P), (L.A_ff, Lo.A_ff), (L.A_fc, Lo.A_fc), (L.A, Lo.A)):
            same(a, o)
    same(H.coarsest_A, Ho.coarsest_A)
    x, st = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig())
    xo, hist, conv, its = O.richardson(Ho, np.zeros(Ao.nrows), np.ones(Ao.nrows))
    assert st.iterations == its
    assert rel(st.residual_history, hist) < 1e-10
    # the device polynomials stay within rounding of the oracle's own
    Hown = O.setup(Ao, O.Cfg(poly_order=order))
    if len(Hown.levels) > 0:
        c_own = Hown.levels[0].smoother.coeffs
        c_dev = H.levels[0].f_smoother.coeffs
        assert len(c_own) == len(c_dev)
        assert np.max(np.abs(c_own - c_dev)) <= 1e-10 * np.max(np.abs(c_own))


def test_neumann_assembly_bitwise(G, hier, hier_hard):
    for h in (hier, hier_hard):
        for L in h.levels[:4]:
            p = O.neumann_poly(L.A_ff, 3)
            same(G.assemble_fixed_sparsity(dev_poly(p), dev_csr(L.A_ff)), O.assemble_poly(p, L.A_ff))


@pytest.mark.parametrize('nx,v', [(48, PI4), (40, HARD)])
def test_krylov_free_setup_bitwise_without_injection(G, nx, v):
    """nAIR variant (Neumann smoothers + Neumann coarse solver, no truncation):
    no Krylov dot products anywhere, so the GPU hierarchy must equal the
    oracle's bit for bit with NO coefficient injection, and the exact-mode
    solve must reproduce x bitwise."""
    kw = dict(inverse_type='neumann', coarsest_inverse_type='neumann', coarsest_poly_order=20,
              auto_truncate_tol=None, poly_order=3, matrix_free_polys=False)
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
    H = G.setup(A, G.SetupConfig(**kw), keep_level_matrices=True)
    Ao = O.advection_2d(nx, nx, *v)
    Ho = O.setup(Ao, O.Cfg(**kw), keep_level_matrices=True)
    assert H.num_levels == len(Ho.levels)
    for L, Lo in zip(H.levels, Ho.levels):
        assert np.array_equal(L.split.labels_host(), Lo.labels)
        for a, o in ((L.R, Lo.R), (L.P, Lo.P), (L.A_ff, Lo.A_ff), (L.A_fc, Lo.A_fc), (L.A, Lo.A),
                     (L.f_smoother_assembled, Lo.assembled)):
            same(a, o)
    same(H.coarsest_A, Ho.coarsest_A)
    x, st = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig(max_iters=60), exact=True)
    xo, hist, conv, its = O.richardson(Ho, np.zeros(Ao.nrows), np.ones(Ao.nrows), max_iters=60)
    assert st.iterations == its
    assert tonp(x).tobytes() == xo.tobytes()


def test_setup_errors(G):
    with pytest.raises(ValueError):
        G.setup(G.SparseMatrix.csr(2, 3, [0, 1, 2], [0, 1], [1.0, 1.0]), G.SetupConfig())
    with pytest.raises(ValueError):
        G.SetupConfig(smooth_type='fcf').validate()
    A = G.build_advection_1d(64, 1.0)
    H = G.setup(A, G.SetupConfig(poly_order=2))
    x, st = G.richardson_solve(H, np.zeros(64), np.ones(64), G.SolveConfig())
    assert st.converged and st.iterations <= 2


@pytest.mark.parametrize('seed,maxlen', [(0, 40), (1, 40), (2, 40), (3, 700), (4, 6)])
def test_ap_onepoint_structural_zeros(G, seed, maxlen):
    """A P for a one-point P (register merge for rows <= 8 / <= 32 entries,
    staged radix sort up to 1024): structure = structural product, values
    summed in A's column order, exact cancellations kept as +0.0 -- bitwise
    the oracle's spgemm(A, P)."""
    import ctypes as C
    import torch
    from paper_2508_17517_b200 import _lib as L
    from paper_2508_17517_b200.csr import take
    rng = np.random.default_rng(seed)
    n, nc = 300, 40
    rows, cols, vals = [], [], []
    if maxlen > n:
        n = 2 * maxlen
    for i in range(n):
        k = int(rng.integers(1, maxlen))
        cs = np.unique(rng.integers(0, n, size=k))
        vs = rng.choice([1.0, -1.0, 0.5, -0.5, 1e-300, 3.0], size=len(cs))
        rows += [i] * len(cs)
        cols += cs.tolist()
        vals += vs.tolist()
    A = O.from_triplets(n, n, np.array(rows), np.array(cols), np.array(vals))
    pcol = rng.integers(0, nc, size=n)
    P = O.from_triplets(n, nc, np.arange(n), pcol, np.ones(n))
    ref = O.spgemm(A, P)
    Ad = dev_csr(A)
    pd = torch.tensor(pcol, dtype=torch.int32, device='cuda')
    res = C.c_void_p()
    L.call('airg_ap_onepoint', n, n, nc, L.ptr(Ad.row_offsets), L.ptr(Ad.col_indices),
           L.ptr(Ad.values), L.ptr(pd), C.byref(res), L.stream_handle())
    same(take(res), ref)
    assert np.any(ref.val == 0.0)          # the case exercises cancellations
    assert not np.any(np.signbit(ref.val[ref.val == 0.0]))


def test_gpu_setup_replayed_by_oracle_512():
    """The benchmark configuration one size down (512^2, default SetupConfig,
    order 6; the reference fixtures stop at 128^2): GPU setup with its own
    device Krylov coefficients, the oracle replays it with those coefficients
    injected.  Every level's labels / R / P / A_ff / A_fc / A and the
    coarsest matrix must be bitwise equal -- this exercises the long-row
    SpGEMM / drop-lump / assembly classes the 2048^2 bench runs (pre-drop
    R(AP) rows up to ~1300 entries) -- and the residual history within
    1e-10 of the initial residual."""
    import paper_2508_17517_b200 as G
    nx = 512
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=PI4[0], vy=PI4[1]))
    H = G.setup(A, G.SetupConfig(), keep_level_matrices=True)
    inj = {k: oracle_poly(p) for k, p in H.polys.items()}
    Ao = O.advection_2d(nx, nx, *PI4)
    Ho = O.setup(Ao, O.Cfg(), poly_inject=inj, keep_level_matrices=True)
    assert H.num_levels == len(Ho.levels)
    assert H.truncated_at == Ho.truncated_at
    for L, Lo in zip(H.levels, Ho.levels):
        assert np.array_equal(L.split.labels_host(), Lo.labels)
        for a, o in ((L.R, Lo.R), (L.P, Lo.P), (L.A_ff, Lo.A_ff), (L.A_fc, Lo.A_fc), (L.A, Lo.A)):
            same(a, o)
    same(H.coarsest_A, Ho.coarsest_A)
    x, st = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig())
    xo, hist, conv, its = O.richardson(Ho, np.zeros(Ao.nrows), np.ones(Ao.nrows))
    assert st.iterations == its
    assert np.max(np.abs(np.array(st.residual_history) - hist)) <= 1e-10 * hist[0]


@pytest.mark.parametrize('order,power', [(6, 1), (40, 1), (6, 3), (6, 6)])
def test_grid_arnoldi_bitwise_multi_kernel(G, order, power):
    """The one-launch cooperative Arnoldi (operators > 1024 rows) computes the
    multi-kernel recurrence with the same per-element assignment and
    reduction order: H, k and beta bitwise equal.  Powers of the stencil
    give 3 / ~10 / ~28 entries per row (1, 2 and 8 SpMV lanes per row)."""
    import os
    from paper_2508_17517_b200.csr import random_unit_vector
    from paper_2508_17517_b200.gmres_poly import hessenberg
    A, _ = G.build_advection_2d(G.AdvectionProblem(nx=120, ny=110, vx=HARD[0], vy=HARD[1]))
    A1 = A
    for _ in range(power - 1):
        A = G.spgemm(A, A1)
    b = random_unit_vector(A.nrows, 3)
    H1, k1, b1 = hessenberg(A, order + 1, b)
    os.environ['AIRG_ARNOLDI_MULTI'] = '1'
    try:
        H2, k2, b2 = hessenberg(A, order + 1, b)
    finally:
        del os.environ['AIRG_ARNOLDI_MULTI']
    assert (k1, b1) == (k2, b2)
    assert H1.tobytes() == H2.tobytes()
