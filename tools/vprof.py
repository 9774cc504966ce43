"""Per-kernel timeline of V-cycles at nx^2 (torch.profiler / CUPTI)."""
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.amg_solve import held_plan
from paper_2508_17517_b200 import _lib as L
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
vx, vy = float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=vx, vy=vy))
H = G.setup(A, G.SetupConfig())
p = held_plan(H)
r = torch.randn(A.nrows, dtype=torch.float64, device='cuda'); e = torch.empty_like(r)
for _ in range(3):
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
    torch.cuda.synchronize()
ev = [x for x in prof.events() if x.device_type.name == 'CUDA']
ev.sort(key=lambda x: x.time_range.start)
per = len(ev) // 5
print('kernels per vcycle', per)
one = ev[per * 2: per * 3]
t0 = one[0].time_range.start
tot = 0
agg = {}
for x in one:
    d = x.time_range.end - x.time_range.start
    tot += d
    k = x.name.split('(')[0][-40:]
    agg[k] = agg.get(k, 0) + d
print('sum kernel us', tot, 'span us', one[-1].time_range.end - t0)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f'{v:9.1f} us  {k}')
print('--- timeline (us: start, dur, name)')
for x in one:
    print(f'{x.time_range.start - t0:8.1f} {x.time_range.end - x.time_range.start:7.1f} {x.name[:60]}')
