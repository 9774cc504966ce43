"""V-cycle time (CUDA events over 20 replays) and roofline fraction at nx^2."""
import sys, os, json
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
for _ in range(5):
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
best = 1e9
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20):
        L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
    e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 20)
by = count_cycle_bytes(H, include_top=False)
print(json.dumps({'env_u': os.environ.get('AIRG_SPMV_U', '4'), 'vcycle_ms': round(best, 4),
                  'GBps': round(by / best / 1e6, 1), 'frac': round(by / best / 1e6 / 6548.2, 4)}))
