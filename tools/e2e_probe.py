"""Where the end-to-end step (host CSR in, x out) spends its time vs the
device-resident step (CUDA events around each part)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
n = A.nrows
G.reserve_memory(n * 1600, n * 4000)
Ap, Ac, Av = (t.cpu().pin_memory() for t in (A.row_offsets, A.col_indices, A.values))
bh = torch.zeros(n, dtype=torch.float64).pin_memory()
xh = torch.ones(n, dtype=torch.float64).pin_memory()
xout = torch.empty(n, dtype=torch.float64).pin_memory()
cfg, scfg = G.SetupConfig(), G.SolveConfig()
x0 = torch.ones(n, dtype=torch.float64, device='cuda')
E = lambda: torch.cuda.Event(enable_timing=True)
res = []
for rep in range(4):
    ev = [E() for _ in range(5)]
    ev[0].record()
    Ad = G.SparseMatrix(n, n, Ap.to('cuda', non_blocking=True), Ac.to('cuda', non_blocking=True),
                        Av.to('cuda', non_blocking=True))
    bd, xd = bh.to('cuda', non_blocking=True), xh.to('cuda', non_blocking=True)
    ev[1].record()
    H = G.setup(Ad, cfg)
    ev[2].record()
    x, _ = G.richardson_solve(H, bd, xd, scfg)
    ev[3].record()
    xout.copy_(x, non_blocking=True)
    ev[4].record()
    torch.cuda.synchronize()
    e2e = [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(4)]
    ev = [E() for _ in range(3)]
    ev[0].record()
    H2 = G.setup(A, cfg)
    ev[1].record()
    x2, _ = G.richardson_solve(H2, b, x0, scfg)
    ev[2].record()
    torch.cuda.synchronize()
    dev = [round(ev[0].elapsed_time(ev[1]), 2), round(ev[1].elapsed_time(ev[2]), 2)]
    res.append({'e2e [h2d, setup, solve, d2h] ms': e2e, 'device [setup, solve] ms': dev})
    del H, H2
print(json.dumps(res[1:]))
