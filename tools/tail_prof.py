"""Host profile of the small-level tail: setup() of the level-L operator of
the 2048^2 hierarchy (default config), cProfile by cumulative and own time."""
import sys, os, cProfile, pstats, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
lev = int(sys.argv[1]) if len(sys.argv) > 1 else 10
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig(), keep_level_matrices=True)
M = H.levels[lev].A
for _ in range(3):
    Hs = G.setup(M, G.SetupConfig())
torch.cuda.synchronize()
t0 = time.perf_counter()
Hs = G.setup(M, G.SetupConfig())
torch.cuda.synchronize()
print(json.dumps({'level': lev, 'n': M.nrows, 'levels': Hs.num_levels,
                  'setup_ms': round(1e3 * (time.perf_counter() - t0), 2),
                  'phases_ms': {k: round(1e3 * x, 2) for k, x in Hs.setup_breakdown.items()}}))
pr = cProfile.Profile()
pr.enable()
Hs = G.setup(M, G.SetupConfig())
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats('cumulative').print_stats(35)
st.sort_stats('tottime').print_stats(20)
