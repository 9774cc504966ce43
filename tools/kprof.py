"""Per-kernel device time of one setup + solve via torch.profiler (CUPTI)."""
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2508_17517_b200 as G
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
order = int(sys.argv[2]) if len(sys.argv) > 2 else 6
vx, vy = float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4))
def step():
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=vx, vy=vy))
    H = G.setup(A, G.SetupConfig(poly_order=order))
    x, st = G.richardson_solve(H, b, torch.ones(A.nrows, dtype=torch.float64, device='cuda'), G.SolveConfig())
    torch.cuda.synchronize()
step()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
agg = {}
for e in prof.events():
    if e.device_type.name != 'CUDA':
        continue
    k = e.name[:90]
    t = e.device_time_total if hasattr(e, 'device_time_total') else e.cuda_time_total
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
print('total_ms', tot / 1e3, 'launches', sum(v[0] for v in agg.values()))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f'{v[1]/1e3:10.2f} ms {v[0]:6d}  {k}')
