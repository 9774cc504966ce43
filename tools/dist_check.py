"""Multi-GPU parity check (run under torchrun, one rank per GPU):
the row-strip distributed setup equals the serial GPU setup bit for bit when
the distributed run's polynomials are injected, and the distributed solve
matches the serial solve's history within 1e-10 of ||r0||.

    torchrun --nproc-per-node 2 tools/dist_check.py [nx] [replicate_below] [weighted]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from tests.gpu_util import tonp
import torch
import torch.distributed as dist


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    rep = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    local = int(os.environ.get('LOCAL_RANK', 0))
    torch.cuda.set_device(local)
    dist.init_process_group('nccl', device_id=torch.device('cuda', local))
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200 import dist as D
    comm = D.Comm()
    v = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))
    cfg = G.SetupConfig(poly_order=4)
    w = None
    if len(sys.argv) > 3 and sys.argv[3] == 'weighted':   # uneven strips
        w = [1.3] + [1.0 + 0.1 * q for q in range(1, comm.world)]
    Ad = D.advection_2d_strips(comm, nx, nx, *v, weights=w)
    DH = D.setup_distributed(comm, Ad, cfg, replicate_below=rep)
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=v[0], vy=v[1]))
    # the generated strips are the global matrix's rows
    full = D.gather_dmat(comm, Ad)
    for x, y in zip(full.to_host(), A.to_host()):
        assert np.array_equal(x, y)
    H = G.setup(A, cfg, poly_inject=DH.polys)
    nd = len(DH.dlevels)
    assert H.num_levels == DH.num_levels, (H.num_levels, DH.num_levels)
    for i, d in enumerate(DH.dlevels):
        L = H.levels[i]
        lab = comm.allgather_v(d.labels)
        assert np.array_equal(lab.cpu().numpy(), L.split.labels_host()), i
        for nm, Md, Ms in (('R', d.R, L.R), ('A_ff', d.A_ff, L.A_ff), ('A_fc', d.A_fc, L.A_fc)):
            dev = Md.values.device
            rows = D.Part.from_counts(comm.allgather_int(Md.nrows), dev)
            g = D.gather_dmat(comm, D.DMat(Md, rows, D.Part([0, Ms.ncols], dev)))
            for x, y in zip(g.to_host(), Ms.to_host()):
                assert x.tobytes() == y.tobytes(), (i, nm)
    for j, L in enumerate(DH.tail.levels):
        Ls = H.levels[nd + j]
        assert np.array_equal(L.split.labels_host(), Ls.split.labels_host())
        for Mt, Ms in ((L.R, Ls.R), (L.A_ff, Ls.A_ff), (L.A_fc, Ls.A_fc)):
            for x, y in zip(Mt.to_host(), Ms.to_host()):
                assert x.tobytes() == y.tobytes()
    for x, y in zip(DH.tail.coarsest_A.to_host(), H.coarsest_A.to_host()):
        assert x.tobytes() == y.tobytes()
    # solve
    S = D.DistSolver(DH)
    lo, hi = Ad.rows.lo(comm.rank), Ad.rows.hi(comm.rank)
    xd, std = S.richardson(torch.zeros(hi - lo, dtype=torch.float64, device='cuda'),
                           torch.ones(hi - lo, dtype=torch.float64, device='cuda'), G.SolveConfig())
    xs, sts = G.richardson_solve(H, b, np.ones(A.nrows), G.SolveConfig())
    hd, hs = np.array(std.residual_history), np.array(sts.residual_history)
    assert std.iterations == sts.iterations, (std.iterations, sts.iterations)
    assert np.max(np.abs(hd - hs)) <= 1e-10 * hs[0], (hd, hs)
    xg = comm.allgather_v(xd).cpu().numpy()
    assert np.max(np.abs(xg - tonp(xs))) <= 1e-9 * np.max(np.abs(tonp(xs))) + 1e-12
    # native plan (C++ V-cycle, NCCL halos, captured graphs)
    for rep in range(2):
        xn, stn = S.solve(torch.zeros(hi - lo, dtype=torch.float64, device='cuda'),
                          torch.ones(hi - lo, dtype=torch.float64, device='cuda'), G.SolveConfig())
        hn = np.array(stn.residual_history)
        assert stn.iterations == sts.iterations, (stn.iterations, sts.iterations)
        assert np.max(np.abs(hn - hs)) <= 1e-10 * hs[0], (hn, hs)
        xg = comm.allgather_v(xn).cpu().numpy()
        assert np.max(np.abs(xg - tonp(xs))) <= 1e-9 * np.max(np.abs(tonp(xs))) + 1e-12
    if comm.rank == 0:
        print(f'DIST OK world={comm.world} nx={nx} dist_levels={nd} total_levels={H.num_levels} '
              f'its={std.iterations} hist_diff={np.max(np.abs(hd - hs)) / hs[0]:.2e}', flush=True)
    dist.destroy_process_group()


if __name__ == '__main__':
    main()
