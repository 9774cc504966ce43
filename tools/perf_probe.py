"""Quick perf probe: setup phases, solve, V-cycle HBM throughput at nx^2."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.amg_solve import held_plan, count_cycle_bytes
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
order = int(sys.argv[2]) if len(sys.argv) > 2 else 6
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
vx, vy = float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4))
for rep in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=vx, vy=vy))
    H = G.setup(A, G.SetupConfig(poly_order=order))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    x, st = G.richardson_solve(H, b, torch.ones(A.nrows, dtype=torch.float64, device='cuda'), G.SolveConfig())
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps({'rep': rep, 'setup_s': t1 - t0, 'solve_s': t2 - t1, 'its': st.iterations,
                      'levels': H.num_levels, 'trunc': H.truncated_at, 'cc': H.cycle_complexity,
                      'breakdown': {k: round(v, 4) for k, v in H.setup_breakdown.items()}}), flush=True)
# V-cycle timing
p = held_plan(H)
r = torch.randn(A.nrows, dtype=torch.float64, device='cuda')
e = torch.empty_like(r)
from paper_2508_17517_b200 import _lib as L
for _ in range(3):
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); ev0.record()
N = 20
for _ in range(N):
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
ev1.record(); torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / N
byts = count_cycle_bytes(H, include_top=False)
print(json.dumps({'vcycle_ms': ms, 'bytes': byts, 'GBps': byts / ms / 1e6, 'frac': byts / ms / 1e6 / 6548.2}))
print(json.dumps(G.hierarchy_summary(H)['levels'][:3]))
