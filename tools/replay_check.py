"""Parity at the benchmarked scale: GPU setup of the nx^2 pi/4 advection
problem (default SetupConfig), then the CPU oracle replays the hierarchy with
the device polynomials injected; every level's labels and
R / P / A_ff / A_fc / A are compared bitwise (sha256 digests) and the solve
histories within 1e-10 of the initial residual.  Writes a JSON summary.

    python tools/replay_check.py 2048 profiles/r02_replay_2048.json
"""
import hashlib, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_17517_b200 as G
from oracle import airg_oracle as O
from tests.gpu_util import host_csr, oracle_poly, tonp


def digest_host(p, c, v):
    h = hashlib.sha256()
    for a in (np.asarray(p, np.int64), np.asarray(c, np.int64), np.asarray(v, np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def dig_dev(M):
    H = host_csr(M)
    return digest_host(H.ptr, H.col, H.val)


def dig_or(M):
    return digest_host(M.ptr, M.col, M.val)


nx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
out = sys.argv[2] if len(sys.argv) > 2 else None
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
t0 = time.time()
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig(), keep_level_matrices=True)
x, st = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig())
gpu_levels = []
for L in H.levels:
    gpu_levels.append({'labels': hashlib.sha256(L.split.labels_host().astype(np.int8).tobytes()).hexdigest(),
                       **{nm: dig_dev(M) for nm, M in (('R', L.R), ('P', L.P), ('A_ff', L.A_ff),
                                                         ('A_fc', L.A_fc), ('A', L.A))}})
gpu_coarsest = dig_dev(H.coarsest_A)
inj = {k: oracle_poly(p) for k, p in H.polys.items()}
t1 = time.time()
Ao = O.advection_2d(nx, nx, *v)
Ho = O.setup(Ao, O.Cfg(), poly_inject=inj, keep_level_matrices=True)
xo, hist, conv, its = O.richardson(Ho, np.zeros(Ao.nrows), np.ones(Ao.nrows))
t2 = time.time()
mism = []
for i, (g, Lo) in enumerate(zip(gpu_levels, Ho.levels)):
    o = {'labels': hashlib.sha256(Lo.labels.astype(np.int8).tobytes()).hexdigest(),
         **{nm: dig_or(M) for nm, M in (('R', Lo.R), ('P', Lo.P), ('A_ff', Lo.A_ff),
                                        ('A_fc', Lo.A_fc), ('A', Lo.A))}}
    for k in o:
        if o[k] != g[k]:
            mism.append(f'level {i} {k}')
if dig_or(Ho.coarsest_A) != gpu_coarsest:
    mism.append('coarsest')
hd = float(np.max(np.abs(np.array(st.residual_history) - hist)) / hist[0])
res = {'nx': nx, 'levels_gpu': H.num_levels, 'levels_oracle': len(Ho.levels),
       'truncated_at': [H.truncated_at, Ho.truncated_at], 'mismatches': mism,
       'bitwise_levels': len(gpu_levels) - len({m.split()[1] for m in mism if m.startswith('level')}),
       'iterations': [st.iterations, its], 'history_maxdiff_rel_r0': hd,
       'x_maxdiff': float(np.max(np.abs(tonp(x) - xo))),
       'gpu_setup_solve_s': round(t1 - t0, 2), 'oracle_replay_s': round(t2 - t1, 1),
       'level_digests_gpu': gpu_levels, 'coarsest_digest': gpu_coarsest}
print(json.dumps({k: res[k] for k in res if k != 'level_digests_gpu'}))
if out:
    json.dump(res, open(out, 'w'), indent=1)
