"""Wall time per libairg entry point, split by setup level (levels >= a
threshold summed), plus the host time between calls.  usage: tail_calls.py [nx] [from_level]"""
import os
import sys
import time

os.environ['AIRG_PROFILE_CALLS'] = '1'
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G
from paper_2508_17517_b200 import _lib as L
from paper_2508_17517_b200 import amg_setup, cfsplit

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
lv0 = int(sys.argv[2]) if len(sys.argv) > 2 else 10
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
state = {'level': -1, 't_level': None}
marks = {}
orig_split = cfsplit.cf_split


def split_hook(*a, **k):
    now = time.perf_counter()
    if state['t_level'] is not None:
        marks[state['level']] = now - state['t_level']
    state['level'] += 1
    state['t_level'] = now
    return orig_split(*a, **k)


amg_setup.cf_split = split_hook  # build_levels imports it per call
cfsplit.cf_split = split_hook
orig_call = L.call
per = {}
per_level = {}


def call_hook(name, *args):
    t0 = time.perf_counter()
    r = orig_call(name, *args)
    if state['level'] >= lv0:
        rec = per.setdefault(name, [0, 0.0])
        rec[0] += 1
        rec[1] += time.perf_counter() - t0
    lvl = per_level.setdefault(state['level'], {})
    lvl[name] = lvl.get(name, 0.0) + time.perf_counter() - t0
    return r


L.call = call_hook
if not os.environ.get('NO_RESERVE'):  # as bench.py: pre-grown pools
    G.reserve_memory(library_bytes=A.nrows * 1600, torch_bytes=A.nrows * 4000)
H = None
for rep in range(3):
    H = None
    per.clear()
    per_level.clear()
    state.update(level=-1, t_level=None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = G.setup(A, G.SetupConfig())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
marks[state['level']] = t1 - state['t_level']
tail = sum(v for k, v in marks.items() if k >= lv0)
calls = sum(v[1] for v in per.values())
print(f'setup {1e3 * (t1 - t0):.1f} ms; levels >= {lv0} (incl. coarse build) wall {1e3 * tail:.1f} ms, '
      f'inside library calls {1e3 * calls:.1f} ms, host between calls {1e3 * (tail - calls):.1f} ms')
print('per level wall (ms):', {k: round(1e3 * v, 2) for k, v in sorted(marks.items())})
for k, v in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print(f'{v[1] * 1e3:8.2f} ms {v[0]:4d} calls  {k}')
top = ['airg_galerkin', 'airg_spgemm', 'airg_poly_assemble', 'airg_arnoldi', 'airg_restriction',
       'airg_ddc_pass', 'airg_cf_pmisr', 'airg_extract']
print('per level, ms in: ' + ' '.join(t[5:] for t in top) + ' other')
for lv in sorted(per_level):
    d = per_level[lv]
    oth = sum(v for k, v in d.items() if k not in top)
    print(f'{lv:>3} ' + ' '.join(f'{1e3 * d.get(t, 0):7.2f}' for t in top) + f' {1e3 * oth:7.2f}')
