"""cProfile of the distributed setup on rank 0 (torchrun)."""
import os, sys, cProfile, pstats, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist


def main():
    local = int(os.environ.get('LOCAL_RANK', 0))
    torch.cuda.set_device(local)
    dist.init_process_group('nccl', device_id=torch.device('cuda', local))
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200 import dist as D
    comm = D.Comm()
    v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    G.reserve_memory(nx * nx * 1600, nx * nx * 4000)
    Ad = D.advection_2d_strips(comm, nx, nx * comm.world, *v)
    for _ in range(2):
        DH = D.setup_distributed(comm, Ad, G.SetupConfig())
    torch.cuda.synchronize(); dist.barrier()
    pr = cProfile.Profile()
    pr.enable()
    DH = D.setup_distributed(comm, Ad, G.SetupConfig())
    torch.cuda.synchronize()
    pr.disable()
    if comm.rank == 0:
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats(os.environ.get('SORT', 'cumulative')).print_stats(45)
        print(s.getvalue()[:9000])
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
