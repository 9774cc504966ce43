"""Time of DistSolver construction vs native plan build vs solve (torchrun)."""
import os, sys, json, time
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
    rows = []
    for rep in range(3):
        DH = D.setup_distributed(comm, Ad, G.SetupConfig())
        ts = []
        for f in (lambda: D.DistSolver(DH), None, None, None):
            torch.cuda.synchronize(); dist.barrier(); t0 = time.perf_counter()
            if f is not None:
                S = f()
            elif len(ts) == 1:
                from paper_2508_17517_b200 import _lib as L
                if L.CALL_TIMES is not None:
                    L.CALL_TIMES.clear()
                S._native()
                if L.CALL_TIMES is not None:
                    torch.cuda.synchronize()
                    calls = {k: [v[0], round(1e3 * v[1], 2)] for k, v in L.CALL_TIMES.items()}
            else:
                S.solve(b, x0, G.SolveConfig())
            torch.cuda.synchronize(); ts.append(round(1e3 * (time.perf_counter() - t0), 2))
        rows.append(ts)
        del S, DH
    if comm.rank == 0:
        print(json.dumps({'world': comm.world, 'ms [DistSolver, native plan, solve1, solve2]': rows}))
        if 'calls' in dir() or True:
            try:
                print(json.dumps(calls))
            except NameError:
                pass
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
