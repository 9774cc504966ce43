"""Hierarchy shape of AIRG on the upwind DG Q1 operator at a few sizes."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
cfgs = json.loads(os.environ.get('DG_CFGS', '[{}]'))
for nx, kw in [(int(a), kw) for a in (sys.argv[1:] or ['64', '128', '256']) for kw in cfgs]:
    A, b = G.build_advection_dg(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    try:
        H = G.setup(A, G.SetupConfig(**kw), keep_level_matrices=True)
    except Exception as e:
        print(json.dumps({'cells': nx, 'cfg': kw, 'error': str(e)[:120]}), flush=True)
        continue
    torch.cuda.synchronize(); t1 = time.perf_counter()
    try:
        x, st = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig())
        its = st.iterations
    except Exception as e:
        its = 'diverged'
    print(json.dumps({'cells': nx, 'cfg': kw, 'its': its, 'n': A.nrows, 'setup_s': round(t1 - t0, 3),
                      'levels': H.num_levels, 'cc': round(H.cycle_complexity, 1),
                      'maxdens': max(round(L.A.nnz / L.n, 1) for L in H.levels)}), flush=True)
