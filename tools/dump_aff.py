"""Dump A_ff of levels 1, 9, 11 of the 2048^2 hierarchy as raw int32/f64 files (tools/micro/chain_bench input)."""
import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2508_17517_b200 as G
nx=2048
v=(float(np.cos(np.pi/4)), float(np.sin(np.pi/4)))
A,b=G.build_advection_2d(G.AdvectionProblem(nx=nx,ny=nx,vx=v[0],vy=v[1]))
H=G.setup(A,G.SetupConfig())
for i in (1, 9, 11):
    M=H.levels[i].A_ff
    M.row_offsets.cpu().numpy().astype(np.int32).tofile(f'gpurun_out/aff{i}_ptr.bin')
    M.col_indices.cpu().numpy().astype(np.int32).tofile(f'gpurun_out/aff{i}_col.bin')
    M.values.cpu().numpy().astype(np.float64).tofile(f'gpurun_out/aff{i}_val.bin')
    print(i, M.nrows, M.nnz if hasattr(M,'nnz') else None)
