"""Column-window statistics of each level's A_ff per SpMV block (256 threads,
VS lanes per row -> 256/VS rows): would staging x[cmin..cmax] in shared
memory pay?  usage: python tools/xwindow_stats.py [nx]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_17517_b200 as G

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
G.reserve_memory(library_bytes=A.nrows * 5600, torch_bytes=A.nrows * 600)
H = G.setup(A, G.SetupConfig())


def pick_vs(mean):
    for t, vs in ((6, 1), (12, 2), (24, 4), (48, 8), (96, 16)):
        if mean <= t:
            return vs
    return 32


for l, lv in enumerate(H.levels):
    for name in ('A_ff', 'R', 'A_fc', 'P'):
        M = getattr(lv, name, None)
        if M is None or M.nrows == 0 or M.nnz == 0:
            continue
        p = M.row_offsets.long()
        c = M.col_indices.long()
        vs = pick_vs(M.nnz / M.nrows)
        rpb = 256 // vs
        nb = (M.nrows + rpb - 1) // rpb
        lens = (p[1:] - p[:-1])
        first = torch.where(lens > 0, c[p[:-1].clamp(max=max(M.nnz - 1, 0))], torch.full_like(lens, 1 << 40))
        last = torch.where(lens > 0, c[(p[1:] - 1).clamp(min=0)], torch.full_like(lens, -1))
        pad = nb * rpb - M.nrows
        first = torch.cat([first, first.new_full((pad,), 1 << 40)]).view(nb, rpb).min(1).values
        last = torch.cat([last, last.new_full((pad,), -1)]).view(nb, rpb).max(1).values
        w = (last - first + 1).clamp(min=0).double()
        q = torch.quantile(w, torch.tensor([0.5, 0.9, 0.99], dtype=torch.float64, device=w.device)).tolist()
        print(f'level {l} {name:4s} rows {M.nrows:8d} nnz/row {M.nnz / M.nrows:6.1f} VS {vs:2d} '
              f'window p50 {q[0]:8.0f} p90 {q[1]:8.0f} p99 {q[2]:8.0f} max {w.max().item():8.0f}  '
              f'sum(window)/nnz {w.sum().item() / M.nnz:6.2f}', flush=True)
