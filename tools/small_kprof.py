"""Kernel time vs wall of setup() on a small coarse operator (CUPTI)."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=2048, ny=2048, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig(), keep_level_matrices=True)
M = H.levels[int(sys.argv[1]) if len(sys.argv) > 1 else 14].A
for _ in range(2):
    G.setup(M, G.SetupConfig())
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    G.setup(M, G.SetupConfig()); torch.cuda.synchronize()
    wall = time.perf_counter() - t0
agg = {}
nk = 0; kt = 0.0; memcpy = 0
for e in prof.events():
    if e.device_type.name != 'CUDA':
        continue
    nk += 1; kt += e.device_time_total
    if 'Memcpy' in e.name: memcpy += 1
    a = agg.setdefault(e.name[:50], [0, 0.0]); a[0] += 1; a[1] += e.device_time_total
top = sorted(([round(v[1] / 1e3, 2), v[0], k] for k, v in agg.items()), reverse=True)[:15]
sync = sum(1 for e in prof.events() if e.name in ('cudaStreamSynchronize', 'cudaDeviceSynchronize', 'cudaEventSynchronize'))
print(json.dumps({'wall_ms': round(1e3 * wall, 2), 'gpu_ops': nk, 'memcpys': memcpy, 'kernel_ms': round(kt / 1e3, 2), 'host_syncs': sync, 'top': top}))
