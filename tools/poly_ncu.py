"""Masked polynomial assembly of one level of the 2048^2 hierarchy inside an
NVTX range "poly" (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
lev = int(sys.argv[1]) if len(sys.argv) > 1 else 8
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A0, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A0, G.SetupConfig(), keep_level_matrices=True)
L = H.levels[lev]
G.assemble_fixed_sparsity(L.f_smoother, L.A_ff)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push('poly')
G.assemble_fixed_sparsity(L.f_smoother, L.A_ff)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
