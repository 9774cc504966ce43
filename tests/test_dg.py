"""Upwind DG (nodal Q1) advection operator, SURVEY 8(d) cfg 5 / BASELINE configs[4].
The reference has no DG generator: oracle.advection_dg_q1 is the
specification (closed-form cell integrals), checked here against 2-point Gauss
quadrature and discrete consistency; the GPU generator must reproduce it bit
for bit, and the AIRG setup on it must be the oracle's (device polynomials
injected)."""

import numpy as np
import pytest

from oracle import airg_oracle as O

PI4 = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))


# ---- CPU: the specification -------------------------------------------------

@pytest.mark.parametrize('v', [PI4, (1.0, 0.0), (0.3, 0.9)])
def test_closed_form_blocks_match_quadrature(v):
    from paper_2508_17517_b200.advection import dg_q1_blocks
    for h in ((1 / 8, 1 / 8), (1 / 5, 1 / 3)):
        spec = dg_q1_blocks(*h, *v)
        quad = O.dg_q1_blocks_gauss(*h, *v)
        for a, b in zip(spec, quad):
            assert np.max(np.abs(a - b)) <= 1e-15


def test_consistency_constant_and_linear_fields():
    nx = ny = 12
    vx, vy = PI4
    A = O.advection_dg_q1(nx, ny, vx, vy).sp()
    h = 1.0 / nx
    e = np.arange(nx * ny)
    i, j = e % nx, e // nx
    interior = (i > 0) & (j > 0)
    # constant field (all nodal values 1): zero residual in interior cells
    r = A @ np.ones(4 * nx * ny)
    for a in range(4):
        assert np.max(np.abs(r[4 * e[interior] + a])) < 1e-15
    # u = x at the nodes: the cell's four rows sum to int_K v . grad u = vx |K|
    k = np.arange(4)
    xs = ((i[:, None] + (k % 2)[None, :]) * h).ravel()
    r = (A @ xs).reshape(-1, 4).sum(axis=1)
    assert np.allclose(r[interior], vx * h * h, rtol=1e-12)


def test_structure():
    A = O.advection_dg_q1(10, 7, *PI4)
    assert A.nrows == 4 * 70
    lens = np.diff(A.ptr)
    assert lens.max() <= 8 and lens.min() >= 4
    # block lower triangular in cell order (upwind neighbours precede)
    rows = np.repeat(np.arange(A.nrows), lens)
    assert np.all(A.col // 4 <= rows // 4)
    assert np.all(A.sp().diagonal() > 0)


# ---- GPU ----------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize('nx,ny,v', [(8, 8, PI4), (33, 17, (0.3, 0.9)), (16, 9, (1.0, 0.0)),
                                     (9, 16, (0.0, 1.0))])
def test_gpu_generator_is_the_spec(nx, ny, v):
    import paper_2508_17517_b200 as G
    A, b = G.build_advection_dg(G.AdvectionProblem(nx=nx, ny=ny, vx=v[0], vy=v[1]))
    spec = O.advection_dg_q1(nx, ny, *v)
    p, c, val = A.to_host()
    assert np.array_equal(p, spec.ptr) and np.array_equal(c, spec.col)
    assert val.tobytes() == spec.val.tobytes()
    assert float(b.abs().max()) == 0.0


@pytest.mark.gpu
def test_airg_on_dg_replayed_by_oracle():
    import paper_2508_17517_b200 as G
    from tests.gpu_util import oracle_poly, host_csr, rel
    nx = 48
    A, b = G.build_advection_dg(G.AdvectionProblem(nx=nx, ny=nx, vx=PI4[0], vy=PI4[1]))
    cfg = G.SetupConfig(poly_order=4)
    H = G.setup(A, cfg, keep_level_matrices=True)
    assert H.num_levels >= 3
    inj = {k: oracle_poly(p) for k, p in H.polys.items()}
    Ao = O.advection_dg_q1(nx, nx, *PI4)
    Ho = O.setup(Ao, O.Cfg(poly_order=4), poly_inject=inj, keep_level_matrices=True)
    assert H.num_levels == len(Ho.levels)
    for L, Lo in zip(H.levels, Ho.levels):
        assert np.array_equal(L.split.labels_host(), Lo.labels)
        for a, o in ((L.R, Lo.R), (L.A_ff, Lo.A_ff), (L.A_fc, Lo.A_fc)):
            h = host_csr(a)
            assert np.array_equal(h.ptr, o.ptr) and np.array_equal(h.col, o.col)
            assert h.val.tobytes() == o.val.tobytes()
    x, st = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig())
    xo, hist, conv, its = O.richardson(Ho, np.zeros(Ao.nrows), np.ones(Ao.nrows))
    assert st.converged and st.iterations == its
    assert rel(st.residual_history, hist) < 1e-10
