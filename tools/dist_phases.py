"""Setup phase times of the distributed setup (rank 0 and the max over
ranks), per level with AIRG_DIST_LEVEL_TIMES=1.  torchrun --nproc-per-node N
tools/dist_phases.py [nx per rank]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault('AIRG_DIST_LEVEL_TIMES', '1')
import numpy as np
import torch
import torch.distributed as dist


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    local = int(os.environ.get('LOCAL_RANK', 0))
    torch.cuda.set_device(local)
    dist.init_process_group('nccl', device_id=torch.device('cuda', local))
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200 import dist as D
    comm = D.Comm()
    v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
    G.reserve_memory(nx * nx * 1600, nx * nx * 4000)
    Ad = D.advection_2d_strips(comm, nx, nx * comm.world, *v)
    DH = None
    for _ in range(3):
        DH = None
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        DH = D.setup_distributed(comm, Ad, G.SetupConfig())
        e1.record()
        torch.cuda.synchronize()
    wall = e0.elapsed_time(e1)
    t = DH.setup_breakdown
    keys = sorted(t)
    vals = torch.tensor([float(t[k]) for k in keys] + [wall], dtype=torch.float64, device='cuda')
    mx = vals.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    if comm.rank == 0:
        print(f'world {comm.world} nx {nx}: setup {wall:.1f} ms (max over ranks {float(mx[-1]):.1f})')
        for i, k in enumerate(keys):
            if '@' not in k and t[k] > 0:
                print(f'  {k:28s} {1e3 * t[k]:8.1f} ms   max {1e3 * float(mx[i]):8.1f}')
        lv = sorted({int(k.split('@')[1]) for k in keys if '@' in k})
        ph = sorted({k.split('@')[0] for k in keys if '@' in k and not k.startswith(('nnz', 'n@'))})
        ph = [p for p in ph if p not in ('nnz_R', 'nnz_AP', 'nnz_Ac', 'n')]
        print('lvl ' + ' '.join(f'{p[-12:]:>12}' for p in ph))
        for l in lv:
            print(f'{l:>3} ' + ' '.join(f'{1e3 * t.get(f"{p}@{l}", 0):12.2f}' for p in ph))
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
