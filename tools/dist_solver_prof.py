"""cProfile of DistSolver construction + first solve on rank 0 (torchrun)."""
import os, sys, cProfile, pstats, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    local = int(os.environ.get('LOCAL_RANK', 0))
    torch.cuda.set_device(local)
    dist.init_process_group('nccl', device_id=torch.device('cuda', local))
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200 import dist as D
    comm = D.Comm()
    v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
    G.reserve_memory(nx * nx * 1600, nx * nx * 4000)
    Ad = D.advection_2d_strips(comm, nx, nx * comm.world, *v)
    n = Ad.M.nrows
    b = torch.zeros(n, dtype=torch.float64, device='cuda')
    x0 = torch.ones(n, dtype=torch.float64, device='cuda')
    for rep in range(3):
        DH = D.setup_distributed(comm, Ad, G.SetupConfig())
        torch.cuda.synchronize(); dist.barrier()
        pr = cProfile.Profile()
        pr.enable()
        S = D.DistSolver(DH)
        S.solve(b, x0, G.SolveConfig())
        torch.cuda.synchronize()
        pr.disable()
        del S, DH
    if comm.rank == 0:
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats('cumulative').print_stats(45)
        print(s.getvalue())
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
