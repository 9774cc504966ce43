"""Does a level's A_ff stay in L2 across the Horner chain?  Times one A_ff
SpMV per level cold (L2 flushed by a 512 MB write before each launch) and
warm (back-to-back repeats), then lists the V-cycle's launches in order with
their durations (CUPTI)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.amg_solve import held_plan
from paper_2508_17517_b200 import _lib as L

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig())
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device='cuda')


def timed(M, x, y, cold, reps=10):
    ts = []
    for _ in range(reps):
        if cold:
            flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        L.call('airg_spmv', M.nrows, L.ptr(M.row_offsets), L.ptr(M.col_indices), L.ptr(M.values),
               L.ptr(x), L.ptr(y), 0, L.stream_handle())
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts[2:]))


rows = []
for i, lv in enumerate(H.levels):
    M = lv.A_ff
    if M.nnz < 200000:
        continue
    x = torch.randn(M.ncols, dtype=torch.float64, device='cuda')
    y = torch.empty(M.nrows, dtype=torch.float64, device='cuda')
    byt = 12 * M.nnz + 4 * (M.nrows + 1) + 8 * M.nrows + 8 * M.ncols
    tc, tw = timed(M, x, y, True), timed(M, x, y, False)
    rows.append(dict(level=i, nnz=M.nnz, mb=round(byt / 1e6, 1), cold_us=round(tc * 1e3, 1),
                     warm_us=round(tw * 1e3, 1), cold_gbs=round(byt / tc / 1e6), warm_gbs=round(byt / tw / 1e6)))
    print(json.dumps(rows[-1]), flush=True)

p = held_plan(H)
r = torch.randn(A.nrows, dtype=torch.float64, device='cuda'); e = torch.empty_like(r)
for _ in range(3):
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
    torch.cuda.synchronize()
evs = sorted([ev for ev in prof.events() if ev.device_type.name == 'CUDA'], key=lambda ev: ev.time_range.start)
for k, ev in enumerate(evs):
    print(k, round(ev.device_time_total, 1), ev.name[:60])
