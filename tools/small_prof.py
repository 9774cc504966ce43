"""cProfile of setup() on a small coarse operator of the 2048^2 hierarchy."""
import sys, os, cProfile, pstats, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200 import _lib as L
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig(), keep_level_matrices=True)
M = H.levels[int(sys.argv[1]) if len(sys.argv) > 1 else 12].A
for _ in range(2):
    G.setup(M, G.SetupConfig())
torch.cuda.synchronize()
if L.CALL_TIMES is not None:
    L.CALL_TIMES.clear()
pr = cProfile.Profile(); pr.enable()
G.setup(M, G.SetupConfig()); torch.cuda.synchronize()
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats('tottime').print_stats(25); print(s.getvalue()[:6000])
if L.CALL_TIMES is not None:
    for k, v in sorted(L.CALL_TIMES.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f'{1e3 * v[1]:8.2f} ms {v[0]:5d}  {k}')
