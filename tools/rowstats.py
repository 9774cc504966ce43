"""Row-length statistics (mean, p99, max) of A_ff, R, A_fc per level of the 2048^2 hierarchy."""
import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2508_17517_b200 as G
nx=2048
v=(float(np.cos(np.pi/4)), float(np.sin(np.pi/4)))
A,b=G.build_advection_2d(G.AdvectionProblem(nx=nx,ny=nx,vx=v[0],vy=v[1]))
H=G.setup(A,G.SetupConfig())
for i,L in enumerate(H.levels):
    for nm in ('A_ff','R','A_fc'):
        M=getattr(L,nm)
        p=M.row_offsets.cpu().numpy(); ln=np.diff(p)
        if len(ln)==0: continue
        # per-CTA max for 148-way split by nnz
        print(i,nm,'n',len(ln),'mean %.1f'%ln.mean(),'p99',int(np.percentile(ln,99)),'max',ln.max())
