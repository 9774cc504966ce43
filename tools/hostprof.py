"""cProfile (host side) of one setup + solve at nx^2."""
import sys, cProfile, pstats, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2508_17517_b200 as G
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
vx, vy = float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4))
def step():
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=vx, vy=vy))
    H = G.setup(A, G.SetupConfig())
    torch.cuda.synchronize()
    return H
step()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable(); H = step(); pr.disable()
print('wall', time.perf_counter() - t0, H.setup_breakdown)
st = pstats.Stats(pr); st.sort_stats('tottime').print_stats(25)
