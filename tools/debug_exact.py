import numpy as np, sys
sys.path.insert(0, '.')
from oracle import airg_oracle as O
from tests.gpu_util import upload_hierarchy, dev_csr, dev_poly
import paper_2508_17517_b200 as G
PI4 = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A = O.advection_2d(64, 64, *PI4)
Hh = O.setup(A, O.Cfg(poly_order=4))
H = upload_hierarchy(Hh)
rng = np.random.default_rng(0)
for lev in range(len(Hh.levels) + 1)[::-1]:
    n = Hh.levels[lev].n if lev < len(Hh.levels) else Hh.coarsest_A.nrows
    r = rng.standard_normal(n)
    want = O.vcycle(Hh, lev, r)
    got = G.vcycle(H, lev, r, G.SolveConfig(), exact=True).cpu().numpy()
    print(lev, n, np.max(np.abs(got - want)), np.isfinite(got).all(), got.tobytes() == want.tobytes())
for L in Hh.levels[:3]:
    b = rng.standard_normal(L.A_ff.nrows)
    want = O.apply_poly(L.smoother, L.A_ff, b)
    got = G.apply_matrix_free(dev_poly(L.smoother), dev_csr(L.A_ff), b, exact=True).cpu().numpy()
    print('poly', np.max(np.abs(got - want)), got.tobytes() == want.tobytes())
    x = rng.standard_normal(L.R.ncols)
    print('spmv', np.array_equal(G.spmv(dev_csr(L.R), x, exact=True).cpu().numpy(), O.spmv(L.R, x)))
