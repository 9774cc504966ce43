"""Wall time per libairg entry point during one setup (AIRG_PROFILE_CALLS=1)."""
import os, sys, time
os.environ['AIRG_PROFILE_CALLS'] = '1'
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200 import _lib as L
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
vx, vy = float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=vx, vy=vy))
H = None
for rep in range(3):
    H = None
    L.CALL_TIMES.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    H = G.setup(A, G.SetupConfig())
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print('rep', rep, 'setup', t1 - t0, {k: round(v, 3) for k, v in H.setup_breakdown.items()})
    ms = torch.cuda.memory_stats()
    print('   torch allocator: device allocs', ms.get('num_device_alloc'), 'frees',
          ms.get('num_device_free'), 'reserved GB', ms.get('reserved_bytes.all.current', 0) / 1e9)
tot = sum(v[1] for v in L.CALL_TIMES.values())
print('sum of call wall', tot)
for k, v in sorted(L.CALL_TIMES.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f'{v[1]*1e3:9.1f} ms {v[0]:5d}  {k}')
