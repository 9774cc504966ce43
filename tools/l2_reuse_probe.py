"""Does L2 (126 MB) serve a level's A_ff on the back-to-back Horner SpMVs?
Times airg_spmv on each level's A_ff cold (after writing a 512 MB buffer)
and warm (right after the same SpMV), CUDA events on the current stream.
usage: python tools/l2_reuse_probe.py [nx]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_17517_b200 as G
from paper_2508_17517_b200.csr import spmv

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
G.reserve_memory(library_bytes=A.nrows * 5600, torch_bytes=A.nrows * 600)
H = G.setup(A, G.SetupConfig())
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
K = 10
if os.environ.get('PROBE_NCU'):  # warm SpMVs of one level inside an NVTX range "probe"
    M = H.levels[int(os.environ['PROBE_NCU'])].A_ff
    x = torch.rand(M.ncols, dtype=torch.float64, device='cuda')
    for _ in range(3):
        spmv(M, x)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push('probe')
    for _ in range(3):
        spmv(M, x)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    sys.exit(0)


def graph_time(fn):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    ts = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts[2:]))


for l, lv in enumerate(H.levels[:12]):
    M = lv.A_ff
    x = torch.rand(M.ncols, dtype=torch.float64, device='cuda')
    mb = (M.nnz * 12 + (M.nrows + 1) * 4 + M.nrows * 8 * 2) / 1e6
    ys = [None]

    def warm():
        for _ in range(K):
            ys[0] = spmv(M, x)

    def cold():
        for _ in range(K):
            flush.fill_(1)
            ys[0] = spmv(M, x)

    def fl():
        for _ in range(K):
            flush.fill_(1)
    tw = graph_time(warm) / K
    tc = (graph_time(cold) - graph_time(fl)) / K
    print(f'level {l}: A_ff {M.nrows} rows {M.nnz} nnz ~{mb:.1f} MB  cold {tc:.1f} us '
          f'({mb / tc:.2f} TB/s)  warm {tw:.1f} us ({mb / tw:.2f} TB/s)', flush=True)
