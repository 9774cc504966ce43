"""cProfile of one warm setup at nx^2: where the host time goes.
usage: setup_cprof.py [nx] [sort]"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
key = sys.argv[2] if len(sys.argv) > 2 else 'tottime'
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
for _ in range(2):
    H = None
    H = G.setup(A, G.SetupConfig())
    torch.cuda.synchronize()
H = None
pr = cProfile.Profile()
pr.enable()
H = G.setup(A, G.SetupConfig())
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats(key).print_stats(30)
