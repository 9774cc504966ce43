"""Per-level setup phase times (CUDA events, H.setup_levels) of a warm
setup at nx^2, and a host-side breakdown of the coarse-solver build.
usage: setup_levels.py [nx]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
if not os.environ.get('NO_RESERVE'):  # as bench.py: pre-grown pools
    G.reserve_memory(library_bytes=A.nrows * 1600, torch_bytes=A.nrows * 4000)
H = None
for rep in range(3):
    H = None  # free the previous hierarchy first (the pool would otherwise grow)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = G.setup(A, G.SetupConfig())
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f'rep {rep}: setup wall {wall * 1e3:.1f} ms, spgemm_coarse '
          f'{H.setup_breakdown["spgemm_coarse"] * 1e3:.1f} ms')
print(f'setup wall {wall * 1e3:.1f} ms; phases (ms):',
      {k: round(v * 1e3, 1) for k, v in H.setup_breakdown.items()})
phases = sorted({p for d in H.setup_levels.values() for p in d})
print('lvl ' + ' '.join(f'{p[:9]:>9}' for p in phases) + '      sum')
tail = 0.0
for lv in sorted(H.setup_levels):
    d = H.setup_levels[lv]
    s = sum(d.values())
    if lv >= 10:
        tail += s
    print(f'{lv:>3} ' + ' '.join(f'{d.get(p, 0) * 1e3:9.2f}' for p in phases) + f' {s * 1e3:8.2f}')
print(f'levels >= 10 (incl. coarsest): {tail * 1e3:.1f} ms')
# coarse solver build, host vs device
from paper_2508_17517_b200.amg_setup import _build_coarse_solver
Cm = H.coarsest_A
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = _build_coarse_solver(Cm, H.config, len(H.levels))
    torch.cuda.synchronize()
    print(f'coarse solver build ({Cm.nrows} rows, order {H.config.coarsest_poly_order}): '
          f'{(time.perf_counter() - t0) * 1e3:.2f} ms')
import cProfile
import pstats
pr = cProfile.Profile()
pr.enable()
s = _build_coarse_solver(Cm, H.config, len(H.levels))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(18)
