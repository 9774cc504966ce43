"""Galerkin R(AP) of one level of the 2048^2 hierarchy in isolation: time,
rows / steps (A entries) / products per output-length class."""
import sys, os, json, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200 import _lib as L
from paper_2508_17517_b200.csr import take
lev = int(sys.argv[1]) if len(sys.argv) > 1 else 5
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A0, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A0, G.SetupConfig(), keep_level_matrices=True)
Lv = H.levels[lev]
A, R = Lv.A, Lv.R
pcol = Lv.P.col_indices if hasattr(Lv, 'P') and Lv.P is not None else None
from paper_2508_17517_b200.amg_setup import _prolong_cols
pcol = _prolong_cols(A, Lv.split)

def galerkin():
    r = C.c_void_p()
    L.call('airg_galerkin', A.nrows, R.nrows, L.ptr(R.row_offsets), L.ptr(R.col_indices),
           L.ptr(R.values), L.ptr(A.row_offsets), L.ptr(A.col_indices), L.ptr(A.values),
           L.ptr(pcol), 1e-6, 1, C.byref(r), L.stream_handle())
    return take(r)
for _ in range(2):
    out = galerkin()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push('rap')
out = galerkin()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    out = galerkin()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
# AP row lengths (after merging): A with columns mapped through pcol
ap = torch.zeros(A.nrows, dtype=torch.int64, device='cuda')
p = A.row_offsets.long(); c = pcol[A.col_indices.long()].long()
rowid = torch.repeat_interleave(torch.arange(A.nrows, device='cuda'), p[1:] - p[:-1])
key = torch.unique(rowid * (R.nrows + 1) + c)
aplen = torch.bincount(key // (R.nrows + 1), minlength=A.nrows)
rp = R.row_offsets.long(); rc = R.col_indices.long()
steps = rp[1:] - rp[:-1]
rrow = torch.repeat_interleave(torch.arange(R.nrows, device='cuda'), steps)
prod = torch.zeros(R.nrows, dtype=torch.int64, device='cuda').index_add_(0, rrow, aplen[rc])
olen = (out.row_offsets[1:] - out.row_offsets[:-1]).long()
res = {'level': lev, 'galerkin_ms': round(ms, 3), 'rows': R.nrows, 'steps': int(steps.sum()),
       'products': int(prod.sum()), 'out_nnz': int(out.nnz)}
for lo, hi, name in ((0, 32, 'c0'), (32, 128, 'c1'), (128, 512, 'c2'), (512, 1024, 'c3'), (1024, 2048, 'c4'), (2048, 10**9, 'c5')):
    m = (olen > lo) & (olen <= hi)  # approximate: classes use the pre-drop length
    res[name] = [int(m.sum()), int(steps[m].sum()), int(prod[m].sum())]
print(json.dumps(res))
