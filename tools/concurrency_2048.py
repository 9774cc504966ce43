"""Two (or more) threads solving on ONE 2048^2 hierarchy on their own streams:
each solve takes its own plan from the hierarchy's pool, so the big
cooperative smoother-chain launches (148 CTAs, ~190 KB of shared memory
each) of the plans run concurrently.  Checks that nothing deadlocks and that
every result is bitwise the single-thread one.  usage: concurrency_2048.py [threads]"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 3
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig())
x0 = torch.ones(A.nrows, dtype=torch.float64, device='cuda')
x_ref, st_ref = G.richardson_solve(H, b, x0, G.SolveConfig())
ref = x_ref.cpu().numpy().tobytes()
out, errs = {}, []


def run(i):
    try:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(4):
                x, st = G.richardson_solve(H, b, x0, G.SolveConfig())
            s.synchronize()
        out[i] = (x.cpu().numpy().tobytes() == ref, st.residual_history == st_ref.residual_history)
    except Exception as e:
        errs.append(repr(e))


t0 = time.time()
th = [threading.Thread(target=run, args=(i,)) for i in range(nt)]
for t in th:
    t.start()
for t in th:
    t.join()
print({'threads': nt, 'errors': errs, 'bitwise': out, 'seconds': round(time.time() - t0, 2)})
assert not errs and all(a and h for a, h in out.values())
print('ok')
