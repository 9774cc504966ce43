"""Serial 2048^2 setup wall time and per-phase breakdown (3 runs, last reported)."""
import sys, os, json, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_17517_b200 as G
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
G.reserve_memory(2048*2048*1600, 2048*2048*4000)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    H = G.setup(A, G.SetupConfig())
    torch.cuda.synchronize(); t1 = time.perf_counter()
print(json.dumps({'serial_setup': round(t1 - t0, 4), 'brk': {k: round(x, 4) for k, x in H.setup_breakdown.items()}}))
