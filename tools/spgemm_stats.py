"""Shape of the setup SpGEMMs on the 2048^2 hierarchy, per level: rows,
products, output entries (pre-drop), column span and column clusters
(maximal runs with gaps < 64) per output row, and the time of each product.
Decides between hash and span-indexed (dense) accumulators."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.amg_setup import _colmaps
from paper_2508_17517_b200.csr import extract_mapped
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A0, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A0, G.SetupConfig(), keep_level_matrices=True)


def prods(A, B):
    p = A.row_offsets.long()
    bl = (B.row_offsets[1:] - B.row_offsets[:-1]).long()
    w = bl[A.col_indices.long()]
    cs = torch.cat([torch.zeros(1, dtype=torch.int64, device='cuda'), torch.cumsum(w, 0)])
    return cs[p[1:]] - cs[p[:-1]]


def stats(M, pr):
    p = M.row_offsets.long(); c = M.col_indices.long()
    lens = p[1:] - p[:-1]
    nz = lens > 0
    first = c[p[:-1][nz]]; last = c[p[1:][nz] - 1]
    span = (last - first + 1).double()
    l = lens[nz].double()
    gap = torch.zeros_like(c, dtype=torch.bool)
    gap[1:] = (c[1:] - c[:-1]) >= 64
    gap[p[:-1][nz]] = True
    rid = torch.repeat_interleave(torch.arange(M.nrows, device='cuda'), lens)
    ncl = torch.zeros(M.nrows, device='cuda', dtype=torch.int64).index_add_(0, rid, gap.long())[nz].double()
    q = lambda t, x: round(float(torch.quantile(t[:16000000].double(), x)), 1) if len(t) else 0
    out = {'rows': M.nrows, 'nnz': M.nnz, 'prod': int(pr.sum()), 'len_mean': round(float(l.mean()), 1),
           'len_p99': q(l, 0.99), 'len_max': int(l.max()) if len(l) else 0,
           'span_mean': round(float(span.mean()), 1), 'span_p99': q(span, 0.99),
           'span_max': int(span.max()) if len(span) else 0,
           'clusters_mean': round(float(ncl.mean()), 1), 'clusters_max': int(ncl.max()) if len(ncl) else 0}
    # entries covered if each row used a dense window of W around its clusters
    for lo, hi in ((0, 128), (128, 512), (512, 1024), (1024, 2048), (2048, 4096), (4096, 1 << 30)):
        m = (l > lo) & (l <= hi)
        if int(m.sum()):
            out[f'L{hi}'] = [int(m.sum()), int(pr[nz][m].sum()), round(float(span[m].mean()), 0),
                             int(span[m].max())]
    return out


def timed(f):
    f(); torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize()
    return r, round((time.perf_counter() - t) * 1e3, 2)


for i, L in enumerate(H.levels):
    A = L.A
    AP, t_ap = timed(lambda: G.spgemm(A, L.P))
    RAP, t_rap = timed(lambda: G.spgemm(L.R, AP))
    fmap, cmap = _colmaps(L.split)
    A_cf = extract_mapped(A, L.split.c_idx, fmap, L.split.n_f)
    Ahat = G.assemble_fixed_sparsity(L.f_smoother, L.A_ff)
    Z, t_z = timed(lambda: G.spgemm(A_cf, Ahat))
    print(json.dumps({'level': i, 'n': A.nrows, 't_ap': t_ap, 't_rap': t_rap, 't_z': t_z,
                      'RAP': stats(RAP, prods(L.R, AP)), 'Z': stats(Z, prods(A_cf, Ahat)),
                      'Aff': stats(L.A_ff, prods(L.A_ff, L.A_ff))}), flush=True)
