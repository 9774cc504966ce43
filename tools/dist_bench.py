"""Weak-scaling timing of the distributed setup + solve (torchrun, 1 rank/GPU).

    torchrun --nproc-per-node N tools/dist_bench.py [nx] [rows_per_rank] [reps] [replicate_below] [force]
"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    per = int(sys.argv[2]) if len(sys.argv) > 2 else 2048   # grid rows per rank
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    rep_below = int(sys.argv[4]) if len(sys.argv) > 4 else 20000
    force = bool(int(sys.argv[5])) if len(sys.argv) > 5 else False
    local = int(os.environ.get('LOCAL_RANK', 0))
    torch.cuda.set_device(local)
    dist.init_process_group('nccl', device_id=torch.device('cuda', local))
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200 import dist as D
    comm = D.Comm()
    ny = per * comm.world
    v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
    G.reserve_memory(nx * per * 1600, nx * per * 4000)
    Ad = D.advection_2d_strips(comm, nx, ny, *v)
    n_loc = Ad.M.nrows
    out, brk = [], None
    for rep in range(reps):
        dist.barrier(); torch.cuda.synchronize(); t0 = time.perf_counter()
        DH = D.setup_distributed(comm, Ad, G.SetupConfig(), replicate_below=rep_below, force=force)
        torch.cuda.synchronize(); dist.barrier(); t1 = time.perf_counter()
        S = D.DistSolver(DH)
        torch.cuda.synchronize(); dist.barrier(); t2 = time.perf_counter()
        x, st = S.solve(torch.zeros(n_loc, dtype=torch.float64, device='cuda'),
                             torch.ones(n_loc, dtype=torch.float64, device='cuda'), G.SolveConfig())
        torch.cuda.synchronize(); dist.barrier(); t3 = time.perf_counter()
        out.append((round(t1 - t0, 4), round(t2 - t1, 4), round(t3 - t2, 4), st.iterations, len(DH.dlevels)))
        brk = {k: round(v, 4) for k, v in DH.setup_breakdown.items() if v}
        del DH, S
    allb = [None] * comm.world
    dist.all_gather_object(allb, brk)
    if comm.rank == 0:
        brk = allb
        print(json.dumps({'world': comm.world, 'grid': [nx, ny], 'replicate_below': rep_below,
                          'runs': out, 'breakdown_last': brk}), flush=True)
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
