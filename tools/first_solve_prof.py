"""Where the first solve of a fresh hierarchy spends its extra time (plan
build, capture preparation, graph capture) vs a cached solve, 2048^2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G
from paper_2508_17517_b200 import _lib as L
from paper_2508_17517_b200.amg_solve import Plan

v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
x0 = torch.ones(A.nrows, dtype=torch.float64, device='cuda')
for rep in range(3):
    H = G.setup(A, G.SetupConfig())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P = Plan(H)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    del P
    t2 = time.perf_counter()
    x, st = G.richardson_solve(H, b, x0, G.SolveConfig())
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    x, st = G.richardson_solve(H, b, x0, G.SolveConfig())
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f'rep {rep}: Plan() {1e3 * (t1 - t0):.2f} ms; first solve {1e3 * (t3 - t2):.2f} ms; '
          f'cached solve {1e3 * (t4 - t3):.2f} ms')
