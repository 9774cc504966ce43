"""Cost of the coarse part of the 2048^2 setup: setup() run on the level-L
operator alone (same config), for a few L."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig(), keep_level_matrices=True)
out = {}
for L in (0, 6, 8, 10, 12, 14):
    M = H.levels[L].A
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        Hs = G.setup(M, G.SetupConfig())
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    out[L] = {'n': M.nrows, 'nnz': M.nnz, 'levels': Hs.num_levels, 'setup_ms': round(1e3 * min(ts), 2)}
print(json.dumps(out))
