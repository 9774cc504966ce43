"""GPU parity of the solve path on identical operators (oracle hierarchy
uploaded to HBM): SpMV, polynomial application, V-cycle and Richardson.

Tolerances: SpMV exact mode is bitwise; the fast (FMA, vector) kernels and
the solve agree with the oracle to 1e-10 relative (north_star tolerance)."""

import numpy as np
import pytest

from oracle import airg_oracle as O
from tests.gpu_util import dev_csr, dev_poly, rel, upload_hierarchy, tonp

pytestmark = pytest.mark.gpu

PI4 = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
HARD = (float(np.sqrt(2 / 3)), float(np.sqrt(1 / 3)))


@pytest.fixture(scope='module')
def G():
    import paper_2508_17517_b200 as G
    return G


@pytest.fixture(scope='module')
def hier64():
    A = O.advection_2d(64, 64, *PI4)
    return O.setup(A, O.Cfg(poly_order=4), keep_level_matrices=True)


def test_spmv_exact_bitwise_on_every_level_operator(G, hier64):
    rng = np.random.default_rng(0)
    mats = [hier64.top_A, hier64.coarsest_A]
    for L in hier64.levels:
        mats += [L.R, L.A_fc, L.A_ff, L.A, L.P]
    for M in mats:
        x = rng.standard_normal(M.ncols)
        want = O.spmv(M, x)
        got = G.spmv(dev_csr(M), x, exact=True).cpu().numpy()
        assert got.tobytes() == want.tobytes()
        fast = G.spmv(dev_csr(M), x).cpu().numpy()
        assert np.allclose(fast, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


def test_spmv_empty_and_ragged(G):
    A = O.from_triplets(5, 7, [0, 0, 3, 3, 3], [1, 6, 0, 2, 5], [1.0, -2.0, 3.0, 0.0, 4.0])
    x = np.arange(7, dtype=np.float64) + 0.5
    assert np.array_equal(G.spmv(dev_csr(A), x, exact=True).cpu().numpy(), O.spmv(A, x))
    Z = O.from_triplets(0, 3, [], [], [])
    assert G.spmv(dev_csr(Z), np.ones(3)).numel() == 0
    with pytest.raises(ValueError):
        G.spmv(dev_csr(A), np.ones(3))


def test_ell_spmv_matches_csr(G, hier64):
    """ELL copy of the structured stencil (and of ragged level operators):
    exact mode bitwise == scipy csr_matvec, fast mode within rounding."""
    from paper_2508_17517_b200.csr import spmv_ell, to_ell
    rng = np.random.default_rng(3)
    A, _ = G.build_advection_2d(G.AdvectionProblem(nx=97, ny=61, vx=PI4[0], vy=PI4[1]))
    E = to_ell(A)
    assert E.width == 3
    x = rng.standard_normal(A.ncols)
    want = O.spmv(O.advection_2d(97, 61, *PI4), x)
    assert spmv_ell(E, x, exact=True).cpu().numpy().tobytes() == want.tobytes()
    assert np.allclose(spmv_ell(E, x).cpu().numpy(), want, rtol=1e-14, atol=1e-14)
    for M in (hier64.levels[2].R, hier64.levels[3].A_ff, hier64.coarsest_A):
        x = rng.standard_normal(M.ncols)
        got = spmv_ell(to_ell(dev_csr(M)), x, exact=True).cpu().numpy()
        assert got.tobytes() == O.spmv(M, x).tobytes()
    with pytest.raises(ValueError):
        to_ell(dev_csr(hier64.levels[2].R), width=1)


def test_poly_apply_kinds_match_oracle(G, hier64):
    rng = np.random.default_rng(1)
    L = hier64.levels[2]
    b = rng.standard_normal(L.A_ff.nrows)
    got = G.apply_matrix_free(dev_poly(L.smoother), dev_csr(L.A_ff), b).cpu().numpy()
    assert rel(got, O.apply_poly(L.smoother, L.A_ff, b)) < 1e-12
    C = hier64.coarsest_A
    bc = rng.standard_normal(C.nrows)
    got = G.apply_matrix_free(dev_poly(hier64.coarse_solver), dev_csr(C), bc).cpu().numpy()
    want = O.apply_poly(hier64.coarse_solver, C, bc)
    assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want))
    nm = O.neumann_poly(L.A_ff, 3)
    got = G.apply_matrix_free(dev_poly(nm), dev_csr(L.A_ff), b).cpu().numpy()
    assert rel(got, O.apply_poly(nm, L.A_ff, b)) < 1e-12


def test_newton_rescale_and_early_exit(G):
    """Wide-spectrum high-order Newton: rescaling / underflow exit semantics
    (polynomial.py:331-353) must match."""
    n = 200
    d = np.linspace(1.0, 1e4, n)
    A = O.from_triplets(n, n, np.arange(n), np.arange(n), d)
    p = O.gmres_poly_newton(A, 80, 3)
    b = np.random.default_rng(2).standard_normal(n)
    want = O.apply_poly(p, A, b)
    got = G.apply_matrix_free(dev_poly(p), dev_csr(A), b).cpu().numpy()
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - want)) <= 1e-9 * np.max(np.abs(want))


def test_vcycle_every_level(G, hier64):
    H = upload_hierarchy(hier64)
    rng = np.random.default_rng(3)
    for lev in range(len(hier64.levels) + 1):
        n = hier64.levels[lev].n if lev < len(hier64.levels) else hier64.coarsest_A.nrows
        r = rng.standard_normal(n)
        want = O.vcycle(hier64, lev, r)
        got = tonp(G.vcycle(H, lev, r, G.SolveConfig()))
        assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want)), lev


@pytest.mark.parametrize('nx,ny,v,order,its', [
    (64, 64, PI4, 4, 1), (128, 128, PI4, 4, 1), (128, 128, PI4, 6, 1), (48, 40, HARD, 6, 1),
    (96, 64, PI4, 3, 2)])
def test_richardson_matches_oracle(G, nx, ny, v, order, its):
    A = O.advection_2d(nx, ny, *v)
    Hh = O.setup(A, O.Cfg(poly_order=order))
    x_o, hist_o, conv_o, its_o = O.richardson(Hh, np.zeros(A.nrows), np.ones(A.nrows),
                                              f_smooth_its=its)
    H = upload_hierarchy(Hh)
    x, st = G.richardson_solve(H, np.zeros(A.nrows), np.ones(A.nrows),
                               G.SolveConfig(f_smooth_its=its))
    assert st.iterations == its_o and st.converged == conv_o
    assert rel(st.residual_history, hist_o) < 1e-10
    x = tonp(x)
    assert np.max(np.abs(x - x_o)) <= 1e-10 * max(np.max(np.abs(x_o)), 1e-300) + 1e-14


@pytest.mark.parametrize('nx,ny,v,order,its', [(64, 64, PI4, 4, 1), (48, 40, HARD, 6, 2)])
def test_richardson_exact_mode_bitwise(G, nx, ny, v, order, its):
    """Parity mode: every kernel follows the reference's arithmetic order, so
    x is bitwise the oracle's (== scipy/numpy) on the same hierarchy."""
    A = O.advection_2d(nx, ny, *v)
    Hh = O.setup(A, O.Cfg(poly_order=order))
    x_o, hist_o, _, its_o = O.richardson(Hh, np.zeros(A.nrows), np.ones(A.nrows),
                                         f_smooth_its=its)
    H = upload_hierarchy(Hh)
    x, st = G.richardson_solve(H, np.zeros(A.nrows), np.ones(A.nrows),
                               G.SolveConfig(f_smooth_its=its), exact=True)
    assert st.iterations == its_o
    assert tonp(x).tobytes() == x_o.tobytes()
    assert rel(st.residual_history, hist_o) < 1e-13
    r = np.random.default_rng(4).standard_normal(A.nrows)
    e = tonp(G.vcycle(H, 0, r, G.SolveConfig(), exact=True))
    assert e.tobytes() == O.vcycle(Hh, 0, r).tobytes()


def test_assembled_smoother_path(G):
    A = O.advection_2d(48, 48, *PI4)
    Hh = O.setup(A, O.Cfg(poly_order=3, matrix_free_polys=False))
    x_o, hist_o, _, its_o = O.richardson(Hh, np.zeros(A.nrows), np.ones(A.nrows))
    H = upload_hierarchy(Hh)
    x, st = G.richardson_solve(H, np.zeros(A.nrows), np.ones(A.nrows), G.SolveConfig())
    assert st.iterations == its_o
    assert rel(st.residual_history, hist_o) < 1e-10


def test_divergence_guard(G):
    A = O.advection_2d(32, 32, *PI4)
    Hh = O.setup(A, O.Cfg(poly_order=2))
    H = upload_hierarchy(Hh)
    bad = O._mk(A.nrows, A.ncols, A.ptr, A.col, -50.0 * A.val)
    H.top_A = dev_csr(bad)
    H._plans = None  # fresh plans for the modified top operator
    with pytest.raises(G.DivergenceError) as ei:
        G.richardson_solve(H, np.zeros(A.nrows), np.ones(A.nrows), G.SolveConfig(max_iters=50))
    assert ei.value.iteration >= 1


def test_solve_bitwise_deterministic(G):
    A = O.advection_2d(64, 64, *PI4)
    H = upload_hierarchy(O.setup(A, O.Cfg(poly_order=4)))
    x1, s1 = G.richardson_solve(H, np.zeros(A.nrows), np.ones(A.nrows), G.SolveConfig())
    x2, s2 = G.richardson_solve(H, np.zeros(A.nrows), np.ones(A.nrows), G.SolveConfig())
    assert s1.residual_history == s2.residual_history
    assert tonp(x1).tobytes() == tonp(x2).tobytes()


def test_concurrent_solves_on_one_hierarchy(G):
    """The reference's Hierarchy is immutable and usable by concurrent solves,
    each owning its work vectors (SPEC.md concurrency model): two threads
    solving on one H on their own streams both reproduce the single-thread
    result bitwise (each solve takes its own plan from H's pool)."""
    import threading
    import torch
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=96, ny=96, vx=PI4[0], vy=PI4[1]))
    H = G.setup(A, G.SetupConfig(poly_order=4))
    x_ref, st_ref = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig())
    out, errs = {}, []

    def run(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    x, st = G.richardson_solve(H, b, np.ones(A.nrows) * (1 + 0 * i),
                                               G.SolveConfig())
                s.synchronize()
            out[i] = (tonp(x), st.residual_history)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        assert out[i][0].tobytes() == tonp(x_ref).tobytes()
        assert out[i][1] == st_ref.residual_history


def test_graph_cache_bounded_and_host_in_host_out(G):
    """vcycle() / richardson_solve() with fresh vectors every call reuse the
    plan's captured graphs (they name the plan's staging vectors), and numpy
    inputs give numpy outputs like the reference's API."""
    from paper_2508_17517_b200 import _lib as L
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=64, ny=64, vx=PI4[0], vy=PI4[1]))
    H = G.setup(A, G.SetupConfig(poly_order=4))
    rng = np.random.default_rng(0)
    for _ in range(40):
        e = G.vcycle(H, 0, rng.standard_normal(A.nrows), G.SolveConfig())
        assert isinstance(e, np.ndarray)
        x, _ = G.richardson_solve(H, b, rng.standard_normal(A.nrows), G.SolveConfig())
        assert isinstance(x, np.ndarray)
    pool = H.__dict__['_plans']
    assert len(pool.all) == 1
    assert L.load().airg_plan_graph_count(pool.all[0].h) <= 4


def test_setup_accepts_reference_style_host_matrix(G):
    """A reference caller's matrix (host CSR with int64 indices, the
    attributes of airmg.SparseMatrix, sparse.py:44-73) is accepted by
    setup() and the sparse kernels, with the same result as the device one."""
    from types import SimpleNamespace
    Ao = O.advection_2d(48, 48, *PI4)
    Ah = SimpleNamespace(nrows=Ao.nrows, ncols=Ao.ncols, row_offsets=Ao.ptr.astype(np.int64),
                         col_indices=Ao.col.astype(np.int64), values=Ao.val)
    H1 = G.setup(Ah, G.SetupConfig(poly_order=4))
    H2 = G.setup(dev_csr(Ao), G.SetupConfig(poly_order=4))
    assert H1.num_levels == H2.num_levels
    for L1, L2 in zip(H1.levels, H2.levels):
        assert np.array_equal(L1.split.labels_host(), L2.split.labels_host())
    y = tonp(G.spmv(Ah, np.ones(Ao.ncols)))
    assert np.max(np.abs(y - O.spmv(Ao, np.ones(Ao.ncols)))) <= 1e-14


@pytest.mark.parametrize('kb,cap', [(64, None), (1, None), (1, 600), (4, 0)])
def test_fused_smoother_chain_partitions(G, hier64, kb, cap, monkeypatch):
    """The fused q(A_ff) chain (chain.cuh) under forced partitions: many CTAs
    (kb: KB of A_ff per CTA), partly staged (cap: staged bytes per CTA) and
    fully unstaged (cap 0) -- the V-cycle stays within 1e-10 of the oracle and
    matches the unfused multi-launch path."""
    monkeypatch.setenv('AIRG_CHAIN', '2')  # every level, whatever its row length
    monkeypatch.setenv('AIRG_CHAIN_KB', str(kb))
    if cap is not None:
        monkeypatch.setenv('AIRG_CHAIN_CAP', str(cap))
    H = upload_hierarchy(hier64)
    rng = np.random.default_rng(5)
    r = rng.standard_normal(hier64.levels[0].n)
    want = O.vcycle(hier64, 0, r)
    got = tonp(G.vcycle(H, 0, r, G.SolveConfig()))
    assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want))
    monkeypatch.setenv('AIRG_CHAIN', '0')
    H2 = upload_hierarchy(hier64)
    ref = tonp(G.vcycle(H2, 0, r, G.SolveConfig()))
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_ell_stencil_path_in_vcycle(G, monkeypatch):
    """ELL copies of the finest level's stencil operators (off by default,
    AIRG_ELL_FILL enables them): the fast-mode solve through the ELL
    epilogue kernel stays within 1e-10 of the oracle."""
    monkeypatch.setenv('AIRG_ELL_FILL', '0.5')
    A = O.advection_2d(80, 72, *PI4)
    Hh = O.setup(A, O.Cfg(poly_order=4))
    x_o, hist_o, conv_o, its_o = O.richardson(Hh, np.zeros(A.nrows), np.ones(A.nrows))
    H = upload_hierarchy(Hh)
    x, st = G.richardson_solve(H, np.zeros(A.nrows), np.ones(A.nrows), G.SolveConfig())
    assert st.iterations == its_o
    assert rel(st.residual_history, hist_o) < 1e-10


def test_concurrent_solves_at_scale_with_cooperative_chains(G):
    """Three threads x four solves on ONE 2048^2 hierarchy: the plans' fused
    smoother chains are cooperative launches of up to 148 CTAs with ~190 KB of
    shared memory each, so concurrent plans cannot be co-resident -- they must
    serialise, not deadlock, and every solve is bitwise the single-thread one."""
    import threading
    import torch
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=PI4[0], vy=PI4[1]))
    H = G.setup(A, G.SetupConfig())
    x0 = torch.ones(A.nrows, dtype=torch.float64, device='cuda')
    x_ref, st_ref = G.richardson_solve(H, b, x0, G.SolveConfig())
    ref = tonp(x_ref).tobytes()
    out, errs = {}, []

    def run(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(4):
                    x, st = G.richardson_solve(H, b, x0, G.SolveConfig())
                s.synchronize()
            out[i] = (tonp(x).tobytes() == ref, st.residual_history == st_ref.residual_history)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th), 'concurrent solves did not finish'
    assert not errs, errs
    assert all(a and h for a, h in out.values()) and len(out) == 3
