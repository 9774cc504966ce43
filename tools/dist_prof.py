"""Kernel timeline of one distributed solve on rank 0 (torchrun)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist


def main():
    rb = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    local = int(os.environ.get('LOCAL_RANK', 0))
    torch.cuda.set_device(local)
    dist.init_process_group('nccl', device_id=torch.device('cuda', local))
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200 import dist as D
    comm = D.Comm()
    v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
    Ad = D.advection_2d_strips(comm, 2048, 2048 * comm.world, *v)
    DH = D.setup_distributed(comm, Ad, G.SetupConfig(), replicate_below=rb)
    S = D.DistSolver(DH)
    n = Ad.M.nrows
    b = torch.zeros(n, dtype=torch.float64, device='cuda')
    x0 = torch.ones(n, dtype=torch.float64, device='cuda')
    S.solve(b, x0, G.SolveConfig())
    torch.cuda.synchronize(); dist.barrier()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        S.solve(b, x0, G.SolveConfig())
        torch.cuda.synchronize()
    if comm.rank == 0:
        ev = sorted([e for e in prof.events() if e.device_type.name == 'CUDA'],
                    key=lambda e: e.time_range.start)
        t0, t1 = ev[0].time_range.start, ev[-1].time_range.end
        agg = {}
        for e in ev:
            k = e.name.split('(')[0][-45:]
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += e.time_range.end - e.time_range.start
        print('span us', t1 - t0, 'kernels', len(ev), 'levels', len(DH.dlevels))
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
            print(f'{t:10.1f} us {c:6d} {k}')
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
