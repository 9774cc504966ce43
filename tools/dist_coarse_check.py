"""configs[3] shape on N ranks: a hierarchy truncated at a low level, so the
coarsest grid is large and solved by the order-100 Newton polynomial.  The
distributed application of that polynomial (DistSolver with the coarsest
operator on row strips) must reproduce the replicated one (AIRG_DIST_COARSE=0)
and the serial solve of the same hierarchy: same iterations, residual
histories within 1e-10 of the initial residual.

    torchrun --nproc-per-node 2 tools/dist_coarse_check.py [nx] [truncate_start]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    start = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    local = int(os.environ.get('LOCAL_RANK', 0))
    torch.cuda.set_device(local)
    dist.init_process_group('nccl', device_id=torch.device('cuda', local))
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200 import dist as D
    comm = D.Comm()
    v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
    cfg = G.SetupConfig(poly_order=4, auto_truncate_start_level=start)
    Ad = D.advection_2d_strips(comm, nx, nx, *v)
    DH = D.setup_distributed(comm, Ad, cfg, replicate_below=500)
    assert DH.tail.num_levels == 0 and DH.truncated_at == start, (DH.tail.num_levels,
                                                                   DH.truncated_at)
    lo, hi = Ad.rows.lo(comm.rank), Ad.rows.hi(comm.rank)
    b = torch.zeros(hi - lo, dtype=torch.float64, device='cuda')
    x0 = torch.ones(hi - lo, dtype=torch.float64, device='cuda')
    hists = {}
    for mode in ('1', '0'):
        os.environ['AIRG_DIST_COARSE'] = mode
        S = D.DistSolver(DH)
        x, st = S.solve(b, x0, G.SolveConfig())
        assert getattr(S, 'dist_coarse', False) == (mode == '1')
        hists[mode] = (st.iterations, np.array(st.residual_history))
        del S
    A, bs = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
    H = G.setup(A, cfg, poly_inject=DH.polys)
    _, sts = G.richardson_solve(H, bs, torch.ones(A.nrows, dtype=torch.float64, device='cuda'),
                                G.SolveConfig())
    hs = np.array(sts.residual_history)
    for mode, (its, h) in hists.items():
        assert its == sts.iterations, (mode, its, sts.iterations)
        assert np.max(np.abs(h - hs)) <= 1e-10 * hs[0], (mode, h, hs)
    if comm.rank == 0:
        n_c = DH.tail.coarsest_A.nrows
        print(f'DIST COARSE OK world={comm.world} nx={nx} coarsest={n_c} '
              f'roots={len(DH.tail.coarse_solver.roots)} its={sts.iterations} '
              f'diff={np.max(np.abs(hists["1"][1] - hs)) / hs[0]:.2e}', flush=True)
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
