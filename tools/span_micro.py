"""R (A P) (plain product) and Z = A_cf Ahat of chosen levels of the 2048^2
hierarchy in isolation: wall time of one call and per-kernel device time
(torch.profiler / CUPTI).  With --nvtx the timed call of the first level is
wrapped in an NVTX range "rap" (ncu target)."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.amg_setup import _colmaps
from paper_2508_17517_b200.csr import extract_mapped
args = [a for a in sys.argv[1:] if not a.startswith('--')]
levels = [int(a) for a in args] or [5, 7]
nvtx = '--nvtx' in sys.argv
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A0, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A0, G.SetupConfig(), keep_level_matrices=True)
from torch.profiler import profile, ProfilerActivity
for a in sys.argv:
    if a.startswith('--kd='):
        os.environ['AIRG_SPAN_KD'] = a[5:]
for lev in levels:
    L = H.levels[lev]
    AP = G.spgemm(L.A, L.P)
    fmap, cmap = _colmaps(L.split)
    A_cf = extract_mapped(L.A, L.split.c_idx, fmap, L.split.n_f)
    Ahat = G.assemble_fixed_sparsity(L.f_smoother, L.A_ff)
    for name, X, Y in (('rap', L.R, AP), ('z', A_cf, Ahat)):
        for _ in range(2):
            G.spgemm(X, Y)
        torch.cuda.synchronize()
        if nvtx and lev == levels[0] and name == 'rap':
            torch.cuda.nvtx.range_push('rap')
        t = time.perf_counter()
        out = G.spgemm(X, Y)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        if nvtx and lev == levels[0] and name == 'rap':
            torch.cuda.nvtx.range_pop()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            G.spgemm(X, Y)
            torch.cuda.synchronize()
        agg = {}
        for e in prof.events():
            if e.device_type.name != 'CUDA':
                continue
            k = e.name.split('(')[0][:60]
            agg[k] = agg.get(k, 0.0) + e.device_time_total / 1e3
        top = {k: round(t, 3) for k, t in sorted(agg.items(), key=lambda kv: -kv[1])[:8]}
        print(json.dumps({'level': lev, 'prod': name, 'ms': round(ms, 2), 'nnz': out.nnz, 'kernels': top}),
              flush=True)
