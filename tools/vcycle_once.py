"""Setup at nx^2, warm V-cycles, then ONE V-cycle inside the NVTX range
"vcycle" (for `ncu --nvtx --nvtx-include vcycle/` DRAM-traffic captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.amg_solve import held_plan, count_cycle_bytes
from paper_2508_17517_b200 import _lib as L
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig())
p = held_plan(H)
r = torch.randn(A.nrows, dtype=torch.float64, device='cuda'); e = torch.empty_like(r)
for _ in range(3):
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
torch.cuda.synchronize()
torch.cuda.nvtx.range_push('vcycle')
L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print('algorithmic_bytes', count_cycle_bytes(H, include_top=False))
