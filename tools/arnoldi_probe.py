"""Time the device Arnoldi (order 7 = poly_order + 1) on A_ff of every level
of the nx^2 hierarchy (configure paths with AIRG_ARNOLDI_* env knobs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G
from paper_2508_17517_b200.csr import random_unit_vector
from paper_2508_17517_b200.gmres_poly import hessenberg

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig())
out = []
tot = 0.0
for i, L in enumerate(H.levels):
    M = L.A_ff
    bb = random_unit_vector(M.nrows, 5)
    hessenberg(M, 7, bb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        hessenberg(M, 7, bb)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5 * 1e3
    tot += dt
    out.append(f'{i}:{M.nrows}:{dt:.2f}')
print(os.environ.get('TAG', ''), f'total {tot:.2f} ms', ' '.join(out))
