import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.amg_solve import held_plan, coarse_mode
from paper_2508_17517_b200 import _lib as L
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
for nx in (512, 1024, 2048):
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
    H = G.setup(A, G.SetupConfig())
    x, st = G.richardson_solve(H, b, torch.ones(A.nrows, dtype=torch.float64, device='cuda'), G.SolveConfig())
    print(nx, H.coarsest_A.nrows, coarse_mode(H), st.iterations)
