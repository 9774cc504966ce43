"""Per-level setup phase times of the nx^2 pi/4 advection hierarchy (CUDA
events on the setup stream, warm second run), plus level sizes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
G.reserve_memory(nx * nx * 1600, nx * nx * 4000)
for _ in range(3):
    H = G.setup(A, G.SetupConfig())
tot = {}
for lev in sorted(H.setup_levels):
    d = H.setup_levels[lev]
    n = H.levels[lev].n if lev < H.num_levels else H.coarsest_A.nrows
    print(json.dumps({'level': lev, 'n': n, 'ms': {k: round(1e3 * x, 2) for k, x in d.items()},
                      'total_ms': round(1e3 * sum(d.values()), 2)}))
    for k, x in d.items():
        tot[k] = tot.get(k, 0) + x
print(json.dumps({'total_ms': {k: round(1e3 * x, 1) for k, x in tot.items()}}))
