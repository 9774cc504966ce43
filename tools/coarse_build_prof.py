"""Timing of the coarse-solver build pieces on the coarsest grid of an
nx^2 hierarchy: device Arnoldi, host root computation, truncation test."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G
from paper_2508_17517_b200.csr import random_unit_vector
from paper_2508_17517_b200.gmres_poly import hessenberg, roots_from_hessenberg, apply_matrix_free

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig())
Cm = H.coarsest_A
bb = random_unit_vector(Cm.nrows, 7)


def tm(f, reps=5):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, r


for env in ('', 'AIRG_ARNOLDI_CTA'):
    if env:
        os.environ[env] = '1'
    t_arn, (Hh, k, beta) = tm(lambda: hessenberg(Cm, 101, bb))
    print(f'Arnoldi order 100 on {Cm.nrows} rows ({env or "warp kernel"}): {t_arn:.2f} ms, k={k}')
    os.environ.pop(env, None)
t_roots, p = tm(lambda: roots_from_hessenberg(Hh, k, beta, 100))
print(f'host roots (harmonic Ritz, Leja, added roots): {t_roots:.2f} ms')
t_app, _ = tm(lambda: apply_matrix_free(p, Cm, bb))
print(f'Newton apply (truncation test): {t_app:.2f} ms')
