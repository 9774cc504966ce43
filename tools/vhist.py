"""Per-launch duration histogram of one V-cycle (torch.profiler / CUPTI)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.amg_solve import held_plan
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
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
    torch.cuda.synchronize()
d = sorted([(ev.device_time_total, ev.name[:40]) for ev in prof.events() if ev.device_type.name == 'CUDA'])
t = np.array([x[0] for x in d])
out = {'n': len(t), 'sum_us': round(t.sum(), 1)}
for lo, hi in ((0, 5), (5, 10), (10, 20), (20, 50), (50, 1e9)):
    m = (t >= lo) & (t < hi)
    out[f'{lo}-{hi}us'] = [int(m.sum()), round(t[m].sum(), 1)]
out['top10'] = [(round(a, 1), b) for a, b in d[-10:]]
print(json.dumps(out))
print('levels', [(L_.n, L_.R.nnz, L_.A_ff.nnz, L_.A_fc.nnz) for L_ in H.levels])
