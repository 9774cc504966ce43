"""Per-kernel device time of the native distributed solve (torchrun); also
solve time vs replicate_below.

    torchrun --nproc-per-node N tools/dist_solve_prof.py [nx] [replicate_below ...]
"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    reps = [int(x) for x in sys.argv[2:]] or [20000]
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
    out = {}
    for rb in reps:
        DH = D.setup_distributed(comm, Ad, G.SetupConfig(), replicate_below=rb)
        S = D.DistSolver(DH)
        S.solve(b, x0, G.SolveConfig())
        ts = []
        for _ in range(5):
            torch.cuda.synchronize(); dist.barrier()
            t0 = time.perf_counter()
            x, st = S.solve(b, x0, G.SolveConfig())
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out[rb] = {'dlevels': len(DH.dlevels), 'levels': DH.num_levels, 'its': st.iterations,
                   'solve_ms': round(1e3 * min(ts), 3)}
        if rb == reps[0]:
            from torch.profiler import profile, ProfilerActivity
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                S.solve(b, x0, G.SolveConfig())
                torch.cuda.synchronize()
            agg = {}
            for e in prof.events():
                if e.device_type.name != 'CUDA':
                    continue
                k = e.name[:60]
                a = agg.setdefault(k, [0, 0.0])
                a[0] += 1
                a[1] += e.device_time_total
            out['kernels'] = sorted(([round(v[1] / 1e3, 3), v[0], k] for k, v in agg.items()),
                                    reverse=True)[:14]
        del DH, S
    if comm.rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
