"""One 2048^2 setup (for ncu captures of setup kernels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig())
torch.cuda.synchronize()
print('levels', H.num_levels, 'breakdown', {k: round(x, 4) for k, x in H.setup_breakdown.items()})
for i, L in enumerate(H.levels):
    print(i, L.n, L.split.n_c, L.R.nnz)
