"""Kernel breakdown (CUPTI) of the Galerkin product R(AP) with drop/lump per
level of the 2048^2 hierarchy: wall ms per call and device ms per kernel.
usage: rap_kernels.py [levels, e.g. 0,1,2,3]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G
from paper_2508_17517_b200 import _lib as L
from paper_2508_17517_b200.amg_setup import _prolong_cols
from paper_2508_17517_b200.csr import take

levels = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else '0,1,2,3').split(',')]
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A0, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A0, G.SetupConfig(), keep_level_matrices=True)
from torch.profiler import ProfilerActivity, profile
for lev in levels:
    Lv = H.levels[lev]
    A, R = Lv.A, Lv.R
    pcol = _prolong_cols(A, Lv.split)

    def galerkin():
        r = C.c_void_p()
        L.call('airg_galerkin', A.nrows, R.nrows, L.ptr(R.row_offsets), L.ptr(R.col_indices),
               L.ptr(R.values), L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
               L.ptr(pcol), 1e-6, 1, C.byref(r), L.stream_handle())
        return take(r)
    for _ in range(2):
        galerkin()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        galerkin()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 3 * 1e3
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        galerkin()
        torch.cuda.synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type.name != 'CUDA':
            continue
        k = e.name.split('(')[0].replace('void ', '').replace('airg::', '')[:44]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    tot = sum(x[1] for x in agg.values())
    print(f'level {lev}: rows {R.nrows} nnz(R) {R.nnz} nnz(A) {A.nnz}: wall {wall:.2f} ms, '
          f'kernel sum {tot / 1e3:.2f} ms')
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:10]:
        print(f'   {t / 1e3:7.3f} ms {c:4d}  {k}')
