import sys; sys.path.insert(0,'.')
import numpy as np, torch, collections
import paper_2508_17517_b200 as G
nx=2048
v=(float(np.cos(np.pi/4)), float(np.sin(np.pi/4)))
A,b=G.build_advection_2d(G.AdvectionProblem(nx=nx,ny=nx,vx=v[0],vy=v[1]))
def step():
    H=G.setup(A,G.SetupConfig())
    x,st=G.richardson_solve(H,b,torch.ones(A.nrows,dtype=torch.float64,device='cuda'),G.SolveConfig())
    torch.cuda.synchronize()
step(); step()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], record_shapes=False, with_stack=True) as prof:
    step()
ev=[e for e in prof.events() if e.device_type.name=='CUDA' and 'Memcpy DtoD' in e.name]
d=sorted([(e.time_range.end-e.time_range.start, e) for e in ev], key=lambda x:-x[0])
print('n', len(ev), 'total us', sum(x[0] for x in d))
for t,e in d[:12]:
    print(round(t,1), e.name)
# CPU-side callers of cudaMemcpyAsync
cpu=[e for e in prof.events() if e.device_type.name=='CPU' and ('aten::copy_' in e.name or 'aten::clone' in e.name)]
c=collections.Counter()
for e in cpu:
    st=[s for s in (e.stack or []) if 'paper_2508' in s]
    c[st[0] if st else 'none']+=1
for k,n in c.most_common(12): print(n, k)
