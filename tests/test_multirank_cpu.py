"""Multi-rank host logic on CPU (gloo, world_size 2): the bench's job time is
the max over ranks, and the reference arm runs on rank 0 only."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(('127.0.0.1', 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR='127.0.0.1', MASTER_PORT=str(port))
    dist.init_process_group('gloo', rank=rank, world_size=world)
    import bench
    got = bench.max_over_ranks(10.0 * (rank + 1), dist, 'cpu')
    out[rank] = got
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert dict(out) == {0: 20.0, 1: 20.0}


def test_reference_arm_nonzero_rank_exits_without_work(capsys):
    import bench

    class A:
        warmup, steps, cpu_nx, order, nx = 1, 1, 16, 2, 16
    assert bench.reference_arm(A, rank=1, world=2) == 0
    assert capsys.readouterr().out == ''


def test_reference_arm_rank0_prints_contract_line(capsys):
    import json
    import bench

    class A:
        warmup, steps, cpu_nx, order, nx = 0, 1, 24, 2, 2048
    assert bench.reference_arm(A, rank=0, world=1) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    for k in ('metric', 'value', 'unit', 'impl', 'cpu_baseline', 'e2e', 'higher_is_better'):
        assert k in line
    assert line['impl'] == 'reference' and line['value'] > 0
    assert line['e2e']['h2d_bytes_per_step'] == 0
    # whole-host time per step: value = sample DOFs / ms_per_step
    n = A.cpu_nx * A.cpu_nx
    assert abs(line['ms_per_step'] - n / line['value'] * 1e3) <= 1e-9 * line['ms_per_step']
    assert line['samples_timed'] >= line['steps']
