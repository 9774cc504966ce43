"""Column span (max - min + 1) vs nnz per row of every coarse operator and R at 2048^2."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig(), keep_level_matrices=True)

def stats(M):
    p = M.row_offsets.long(); c = M.col_indices.long()
    n = M.nrows
    lens = p[1:] - p[:-1]
    nz = lens > 0
    first = c[p[:-1][nz]]; last = c[p[1:][nz] - 1]
    span = (last - first + 1).double()
    l = lens[nz].double()
    q = lambda t, x: float(torch.quantile(t[:min(len(t), 16000000)], x)) if len(t) else 0
    return {'rows': n, 'nnz/row': round(float(l.mean()), 1), 'span mean': round(float(span.mean()), 1),
            'span p50': q(span, 0.5), 'span p99': q(span, 0.99), 'span max': float(span.max()),
            'span/nnz': round(float((span / l).mean()), 2)}

out = []
for i, L in enumerate(H.levels):
    Ac = H.levels[i + 1].A if i + 1 < len(H.levels) else H.coarsest_A
    out.append({'level': i, 'Ac': stats(Ac), 'R': stats(L.R)})
for o in out:
    print(json.dumps(o))
