"""The row-strip distributed path (dist.py + the airg_dplan plan) on the GPU.

* one GPU: the distributed code path forced on a single NCCL rank must build
  the serial hierarchy bit for bit (same polynomials injected) and its native
  solve must reproduce the serial history within 1e-10 of ||r0||;
* two GPUs (skipped on smaller boxes): tools/dist_check.py under torchrun —
  the same checks across real row strips with NVLink peer-store halos.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PI4 = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))


def _free_port():
    s = socket.socket()
    s.bind(('127.0.0.1', 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope='module')
def single_rank():
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR='127.0.0.1', MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group('nccl', rank=0, world_size=1, device_id=torch.device('cuda', 0))
    yield dist
    dist.destroy_process_group()


def _bytes_equal(Md, Ms):
    for x, y in zip(Md.to_host(), Ms.to_host()):
        assert x.tobytes() == y.tobytes()


def test_distributed_path_on_one_rank_is_the_serial_hierarchy(single_rank):
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200 import dist as D
    comm = D.Comm()
    cfg = G.SetupConfig(poly_order=4)
    nx = 96
    Ad = D.advection_2d_strips(comm, nx, nx, *PI4)
    DH = D.setup_distributed(comm, Ad, cfg, replicate_below=800, force=True)
    assert len(DH.dlevels) >= 3
    A, b = G.build_advection_2d(G.AdvectionProblem(nx=nx, ny=nx, vx=PI4[0], vy=PI4[1]))
    _bytes_equal(Ad.M, A)
    H = G.setup(A, cfg, poly_inject=DH.polys)
    assert H.num_levels == DH.num_levels
    for i, d in enumerate(DH.dlevels):
        L = H.levels[i]
        assert np.array_equal(d.labels.cpu().numpy(), L.split.labels_host())
        _bytes_equal(d.R, L.R)
        _bytes_equal(d.A_ff, L.A_ff)
        _bytes_equal(d.A_fc, L.A_fc)
    nd = len(DH.dlevels)
    for j, L in enumerate(DH.tail.levels):
        _bytes_equal(L.R, H.levels[nd + j].R)
    _bytes_equal(DH.tail.coarsest_A, H.coarsest_A)
    # native distributed solve vs the serial solve
    S = D.DistSolver(DH)
    n = A.nrows
    xd, sd = S.solve(torch.zeros(n, dtype=torch.float64, device='cuda'),
                     torch.ones(n, dtype=torch.float64, device='cuda'), G.SolveConfig())
    xs, ss = G.richardson_solve(H, b, torch.ones(n, dtype=torch.float64, device='cuda'),
                                G.SolveConfig())
    hd, hs = np.array(sd.residual_history), np.array(ss.residual_history)
    assert sd.iterations == ss.iterations
    assert np.max(np.abs(hd - hs)) <= 1e-10 * hs[0]
    assert torch.max(torch.abs(xd - xs)).item() <= 1e-9 * torch.max(torch.abs(xs)).item() + 1e-12


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason='needs two GPUs')
def test_two_gpu_strips_match_serial():
    cmd = [sys.executable, '-m', 'torch.distributed.run', '--nnodes=1', '--nproc-per-node', '2',
           '--master-addr', '127.0.0.1', '--master-port', str(_free_port()),
           os.path.join(ROOT, 'tools', 'dist_check.py'), '192', '1500', 'weighted']
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=420)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert 'DIST OK world=2' in r.stdout + r.stderr


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 4,
                    reason='needs four GPUs')
def test_four_gpu_strips_match_serial():
    """4 ranks: the coarse levels couple non-adjacent strips; hierarchy bitwise
    the serial one under injection, solve within 1e-10 (tools/dist_check.py)."""
    cmd = [sys.executable, '-m', 'torch.distributed.run', '--nnodes=1', '--nproc-per-node', '4',
           '--master-addr', '127.0.0.1', '--master-port', str(_free_port()),
           os.path.join(ROOT, 'tools', 'dist_check.py'), '256', '1500', 'weighted']
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert 'DIST OK world=4' in r.stdout + r.stderr


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason='needs two GPUs')
def test_two_gpu_distributed_newton_coarse():
    """configs[3] shape at 2 ranks: truncation at level 2 leaves a coarsest grid
    of ~10k rows solved by the order-100 Newton polynomial.  Its distributed
    application (row strips, ghost exchange per SpMV, one max-allreduce per
    root) must give the same residual history as the replicated one."""
    cmd = [sys.executable, '-m', 'torch.distributed.run', '--nnodes=1', '--nproc-per-node', '2',
           '--master-addr', '127.0.0.1', '--master-port', str(_free_port()),
           os.path.join(ROOT, 'tools', 'dist_coarse_check.py'), '256', '3']
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=420)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert 'DIST COARSE OK world=2' in r.stdout + r.stderr
