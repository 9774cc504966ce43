"""B-row sharing if 2/4/8 adjacent Galerkin output rows were walked together: union of their R-row columns / sum of lengths, per level."""
import sys; sys.path.insert(0,'.')
import numpy as np, scipy.sparse as sp
import paper_2508_17517_b200 as G
nx=int(sys.argv[1]) if len(sys.argv)>1 else 2048
v=(float(np.cos(np.pi/4)), float(np.sin(np.pi/4)))
A,b=G.build_advection_2d(G.AdvectionProblem(nx=nx,ny=nx,vx=v[0],vy=v[1]))
H=G.setup(A,G.SetupConfig())
for i,L in enumerate(H.levels[:12]):
    R=L.R
    p=R.row_offsets.cpu().numpy(); c=R.col_indices.cpu().numpy()
    m=len(p)-1
    M=sp.csr_matrix((np.ones(len(c),dtype=np.int8),c,p),shape=(m,L.n))
    tot=M.nnz
    # also the B = AP rows touched: same k set (row k of AP for k in R row)
    out=[f'level {i} m {m} nnz(R) {tot}']
    for g in (2,4,8):
        q=(m+g-1)//g
        S=sp.csr_matrix((np.ones(m,dtype=np.int32),np.arange(m)//g,np.arange(m+1)),shape=(m,q)).T.tocsr()
        U=(S@M); U.data[:]=1
        out.append(f'g{g}: loads/row-load {U.nnz/tot:.3f}')
    print('  '.join(out), flush=True)
