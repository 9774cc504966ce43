"""Cost of the coarsest-level work of the 2048^2 hierarchy: order-100 Newton
polynomial (device Arnoldi, host roots) and the truncation test."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.csr import random_unit_vector
from paper_2508_17517_b200.gmres_poly import hessenberg, roots_from_hessenberg
from paper_2508_17517_b200.amg_setup import try_truncate, derive_seed
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A0, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A0, G.SetupConfig())
C = H.coarsest_A


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
    torch.cuda.synchronize()
    return r, round((time.perf_counter() - t0) / reps * 1e3, 3)


bb = random_unit_vector(C.nrows, 7)
(Hh, k, beta), t_arn = t(lambda: hessenberg(C, 101, bb))
_, t_roots = t(lambda: roots_from_hessenberg(Hh, k, beta, 100))
_, t_newton = t(lambda: G.gmres_poly_newton(C, 100, 7))
_, t_trunc = t(lambda: try_truncate(C, G.SetupConfig(), 18, start_level=0))
print(json.dumps({'n': C.nrows, 'nnz': C.nnz, 'arnoldi_ms': t_arn, 'roots_ms': t_roots,
                  'newton_total_ms': t_newton, 'try_truncate_ms': t_trunc}))
