"""Per-(level, operation) device time and bandwidth of one fast-mode V-cycle.

Launch order of vcycle_rec (solve.cu) with fits=1 and coefficient smoothers:
R_0 .. R_{L-1}, coarse, then for l = L-1 .. 0: A_fc (+ e[c] scatter), d Horner
steps (d=0: one axpby).  Each launch gets its algorithmic bytes from the same
model as count_cycle_bytes; durations are the median over repeated V-cycles
(CUPTI via torch.profiler, graph-replayed).  usage: vlevels.py [nx] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_17517_b200 as G
from paper_2508_17517_b200 import _lib as L
from paper_2508_17517_b200.amg_solve import _spmat_bytes, held_plan

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 9
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
H = G.setup(A, G.SetupConfig())
p = held_plan(H)
r = torch.randn(A.nrows, dtype=torch.float64, device='cuda')
e = torch.empty_like(r)
for _ in range(3):
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
torch.cuda.synchronize()

from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof0:
    L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
    torch.cuda.synchronize()
names = [x.name for x in sorted(prof0.events(), key=lambda x: x.time_range.start)
         if x.device_type.name == 'CUDA' and not x.name.startswith('Memcpy')]

ops = []
for li, lv in enumerate(H.levels):
    ops.append((li, 'R', _spmat_bytes(lv.R) + 8 * lv.n + 8 * lv.split.n_c))
Cm = H.coarsest_A
ops.append((len(H.levels), 'coarse', 8 * Cm.nrows * Cm.nrows + 16 * Cm.nrows))
for li in range(len(H.levels) - 1, -1, -1):
    lv = H.levels[li]
    nf, nc = lv.split.n_f, lv.split.n_c
    d = len(lv.f_smoother.coeffs) - 1
    fused0 = d == 0 and (len(ops) + 1 >= len(names) or 'axpby' not in names[len(ops) + 1])
    if fused0:  # degree 0: e[f] = c0 (r[f] - A_fc e_c) in the A_fc launch
        ops.append((li, 'Afc+e', _spmat_bytes(lv.A_fc) + 24 * nc + 16 * nf))
        continue
    ops.append((li, 'Afc', _spmat_bytes(lv.A_fc) + 8 * nc + 16 * nf + 16 * nc))
    if d == 0:
        ops.append((li, 'axpby', 24 * nf))
    elif 'chain_kernel' in names[len(ops)]:  # fused chain: one launch, the same (unfused) byte model
        ops.append((li, 'H', d * (_spmat_bytes(lv.A_ff) + 24 * nf)))
    else:
        for j in range(d):
            ops.append((li, f'H{j}', _spmat_bytes(lv.A_ff) + 24 * nf))

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        L.call('airg_plan_vcycle', p.h, 0, L.ptr(r), L.ptr(e), 1, L.stream_handle())
    torch.cuda.synchronize()
ev = [x for x in prof.events() if x.device_type.name == 'CUDA' and not x.name.startswith('Memcpy')]
ev.sort(key=lambda x: x.time_range.start)
per = len(ev) // reps
if per != len(ops):
    print(f'launch count {per} != modelled {len(ops)}; names:', [x.name[:30] for x in ev[:per]])
    sys.exit(1)
dur = np.array([[ev[k * per + i].time_range.end - ev[k * per + i].time_range.start
                 for i in range(per)] for k in range(reps)])
span = np.array([ev[k * per + per - 1].time_range.end - ev[k * per].time_range.start
                 for k in range(reps)])
med = np.median(dur, axis=0)
gaps = np.median(np.array([[max(0.0, ev[k * per + i].time_range.start - ev[k * per + i - 1].time_range.end)
                            for i in range(1, per)] for k in range(reps)]), axis=0)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   'MEASURED_PEAKS.json')))
peak = float(peak.get('hbm_gbs', 6458.4))
rows = []
agg = {}
for (li, op, by), t in zip(ops, med):
    rows.append({'level': li, 'op': op, 'us': round(float(t), 2), 'MB': round(by / 1e6, 3),
                 'GBps': round(by / t / 1e3, 1)})
    key = (li, op[0] if op.startswith('H') else op)
    a = agg.setdefault(key, [0.0, 0])
    a[0] += t
    a[1] += by
tot_b = sum(o[2] for o in ops)
print(json.dumps({'nx': nx, 'launches': per, 'span_us_median': float(np.median(span)),
                  'kernel_sum_us': float(med.sum()), 'gap_sum_us': float(gaps.sum()), 'bytes': tot_b,
                  'frac_span': tot_b / (np.median(span) * 1e-6) / (peak * 1e9)}))
print(f'{"lvl":>3} {"op":>6} {"us":>8} {"MB":>9} {"GB/s":>8} {"frac":>6}')
for (li, op), (t, by) in sorted(agg.items()):
    print(f'{li:>3} {op:>6} {t:8.1f} {by / 1e6:9.2f} {by / t / 1e3:8.0f} {by / t / 1e3 / peak:6.2f}')
small = med < 10
print('launches < 10us:', int(small.sum()), 'sum', round(float(med[small].sum()), 1), 'us')
json.dump(rows, open(os.environ.get('VLEVELS_OUT', '/dev/null'), 'w'))
