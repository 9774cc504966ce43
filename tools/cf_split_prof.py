"""Host wall time of cf_split and its library calls on small levels (the
setup tail is latency-bound).  usage: python tools/cf_split_prof.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200 import cfsplit as CS
from paper_2508_17517_b200.cfsplit import F_POINT
from paper_2508_17517_b200.csr import as_matrix


def timeit(f, reps=50):
    f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


for nx in (32, 64, 256, 1024):
    v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
    A = as_matrix(G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))[0])
    row = {'n': A.nrows}
    row['cf_split'] = timeit(lambda: CS.cf_split(A, 0.5, 0.1, 2, 7))
    lab = CS._cf_labels(A, 0.5, 7)
    row['cf_labels'] = timeit(lambda: CS._cf_labels(A, 0.5, 7))
    row['item'] = timeit(lambda: int((lab == F_POINT).sum().item()))
    row['ddc_pass'] = timeit(lambda: CS._ddc_labels(A, lab.clone(), 0.1, 1000))
    row['clone'] = timeit(lambda: lab.clone())
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in row.items()}, flush=True)

if os.environ.get('KPROF'):
    from torch.profiler import profile, ProfilerActivity
    for nx in (32, 1024):
        v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
        A = as_matrix(G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))[0])
        lab = CS._cf_labels(A, 0.5, 7)
        CS._ddc_labels(A, lab.clone(), 0.1, 1000)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            for _ in range(5):
                CS._ddc_labels(A, lab.clone(), 0.1, 1000)
            torch.cuda.synchronize()
        print(nx, prof.key_averages().table(sort_by='cuda_time_total', row_limit=14), flush=True)
