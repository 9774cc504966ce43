"""Device kernel time vs wall time of one distributed setup, per rank (torchrun)."""
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
    for _ in range(2):
        D.setup_distributed(comm, Ad, G.SetupConfig())
    from torch.profiler import profile, ProfilerActivity
    torch.cuda.synchronize(); dist.barrier()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        DH = D.setup_distributed(comm, Ad, G.SetupConfig())
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    agg, tot, nccl = {}, 0.0, 0.0
    for e in prof.events():
        if e.device_type.name != 'CUDA':
            continue
        k = e.name[:50]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.device_time_total
        tot += e.device_time_total
        if 'nccl' in k:
            nccl += e.device_time_total
    top = sorted(([round(v[1] / 1e3, 2), v[0], k] for k, v in agg.items()), reverse=True)[:12]
    res = {'rank': comm.rank, 'wall_s': round(wall, 3), 'device_ms': round(tot / 1e3, 1),
           'nccl_ms': round(nccl / 1e3, 1), 'launches': sum(v[0] for v in agg.values()), 'top': top}
    out = [None] * comm.world
    dist.all_gather_object(out, res)
    if comm.rank == 0:
        for r in out:
            print(json.dumps(r))
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
