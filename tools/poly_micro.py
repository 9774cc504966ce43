"""Polynomial phase of chosen levels of the 2048^2 hierarchy, split into
device Arnoldi, host coefficient algebra and the masked assembly."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.csr import random_unit_vector
from paper_2508_17517_b200.gmres_poly import hessenberg, coeffs_from_hessenberg
levels = [int(a) for a in sys.argv[1:]] or [1, 5, 8]
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A0, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A0, G.SetupConfig(), keep_level_matrices=True)


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
    torch.cuda.synchronize()
    return r, round((time.perf_counter() - t0) / reps * 1e3, 3)


for lev in levels:
    Aff = H.levels[lev].A_ff
    bb = random_unit_vector(Aff.nrows, 5)
    (Hh, k, beta), t_arn = t(lambda: hessenberg(Aff, 7, bb))
    _, t_coef = t(lambda: coeffs_from_hessenberg(Hh, k, beta, 6))
    p = H.levels[lev].f_smoother
    _, t_asm = t(lambda: G.assemble_fixed_sparsity(p, Aff))
    print(json.dumps({'level': lev, 'n_f': Aff.nrows, 'nnz_Aff': Aff.nnz, 'arnoldi_ms': t_arn,
                      'coeffs_ms': t_coef, 'assembly_ms': t_asm}), flush=True)
