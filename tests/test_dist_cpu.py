"""Host-side exchange logic of the row-strip decomposition (dist.py) on CPU:
gloo, world_size 2.  Partitions, ghost-value halos, ghost-row fetches and the
in-place [local | ghost] column renumbering are checked against the global
objects every rank can build itself."""

import os
import socket

import numpy as np
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


def _global_csr(n, seed=3, kmax=6):
    """A random global CSR (sorted columns, every row non-empty)."""
    rng = np.random.default_rng(seed)
    ptr, col, val = [0], [], []
    for i in range(n):
        k = int(rng.integers(1, kmax))
        c = np.unique(np.concatenate([[i], rng.integers(0, n, size=k)]))
        col.extend(c.tolist())
        val.extend((1000.0 * i + c).tolist())
        ptr.append(len(col))
    return np.array(ptr), np.array(col), np.array(val)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR='127.0.0.1', MASTER_PORT=str(port))
    dist.init_process_group('gloo', rank=rank, world_size=world)
    try:
        from paper_2508_17517_b200 import dist as D
        from paper_2508_17517_b200.csr import SparseMatrix
        cpu = torch.device('cpu')
        comm = D.Comm(device=cpu)
        # uneven strips (world 2: 17 + 20 rows; world 8: 5..16 rows)
        counts = [17, 20] if world == 2 else [5 + (3 * r) % 12 for r in range(world)]
        n = sum(counts)
        part = D.Part.from_counts(counts, cpu)
        lo, hi = part.lo(rank), part.hi(rank)
        # owner lookup
        g = torch.arange(n)
        assert part.owner(g).tolist() == sum(([r] * c for r, c in enumerate(counts)), [])
        # collectives
        assert comm.allgather_int(rank + 5) == [5 + r for r in range(world)]
        assert comm.sum_int(rank + 1) == world * (world + 1) // 2
        v = torch.arange(lo, hi, dtype=torch.float64)
        assert comm.allgather_v(v).tolist() == list(range(n))
        # the global matrix; this rank's rows with global column ids (columns
        # drawn from the whole range: every rank couples to every other, the
        # all-to-all pattern of the coarse levels at 8 ranks)
        P, C, V = _global_csr(n, kmax=6 if world == 2 else 14)
        lp = torch.tensor(P[lo:hi + 1] - P[lo], dtype=torch.int32)
        lc = torch.tensor(C[P[lo]:P[hi]], dtype=torch.int32)
        lv = torch.tensor(V[P[lo]:P[hi]], dtype=torch.float64)
        M = SparseMatrix(hi - lo, n, lp, lc, lv)
        need = D.remote_cols(M.col_indices, part, rank)
        if world == 8:  # the case exercises all-to-all couplings
            assert set(part.owner(need).tolist()) == set(range(world)) - {rank}
        expect_need = sorted({int(c) for c in lc.tolist() if not lo <= c < hi})
        assert need.tolist() == expect_need
        halo = D.Halo(comm, part, need)
        # ghost values: every rank's local value of global id i is 0.5 * i
        local = 0.5 * torch.arange(lo, hi, dtype=torch.float64)
        assert halo.values(local).tolist() == [0.5 * i for i in expect_need]
        ext = halo.ext(local)
        # renumbering keeps the stored order and maps to [local | ghost]
        xc = halo.ext_cols(M.col_indices)
        glob_of_ext = torch.cat([torch.arange(lo, hi), torch.tensor(expect_need, dtype=torch.int64)])
        assert glob_of_ext[xc.long()].tolist() == lc.tolist()
        # y = M x computed with ghosts equals the global product's rows
        y = torch.zeros(hi - lo, dtype=torch.float64)
        for i in range(hi - lo):
            for k in range(int(lp[i]), int(lp[i + 1])):
                y[i] += lv[k] * ext[xc[k]]
        full = np.zeros(n)
        for i in range(n):
            full[i] = sum(V[k] * 0.5 * C[k] for k in range(P[i], P[i + 1]))
        assert np.array_equal(y.numpy(), full[lo:hi])
        # ghost ROWS: the rows of the remote ids, exactly as stored globally
        gp, gc, gv = halo.rows(M)
        for j, gid in enumerate(expect_need):
            a, b = int(gp[j]), int(gp[j + 1])
            assert gc[a:b].tolist() == C[P[gid]:P[gid + 1]].tolist()
            assert gv[a:b].tolist() == V[P[gid]:P[gid + 1]].tolist()
        # local rows followed by ghost rows
        R = D.cat_rows(M, gp, gc, gv, n)
        assert R.nrows == (hi - lo) + len(expect_need)
        # batched plans (one all-gather + one all-to-all) == one plan per item
        part2 = D.Part.from_counts([30, 7] if world == 2 else counts[::-1], cpu)
        rng = np.random.default_rng(11 + rank)
        lo2, hi2 = part2.lo(rank), part2.hi(rank)
        need2 = torch.tensor(sorted({int(c) for c in rng.integers(0, n, 25)
                                     if not lo2 <= c < hi2}), dtype=torch.int64)
        items = [(part, need), (part2, need2), (part, torch.zeros(0, dtype=torch.int64)),
                 (part2, need2[:3])]
        single = [D.Halo(comm, p_, q_) for p_, q_ in items]
        batch = D.Halo.many(comm, items)
        for s_, b_ in zip(single, batch):
            assert s_.n == b_.n and s_.n_loc == b_.n_loc
            assert list(s_.recv_counts) == list(b_.recv_counts)
            assert list(s_.send_counts) == list(b_.send_counts)
            assert s_.send_idx.tolist() == b_.send_idx.tolist()
            loc2 = 0.25 * torch.arange(b_.part.lo(rank), b_.part.hi(rank), dtype=torch.float64)
            assert b_.values(loc2).tolist() == s_.values(loc2).tolist()
        out[rank] = 'ok'
    except Exception as e:  # surface the failing assertion in the parent
        import traceback
        out[rank] = traceback.format_exc()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize('world', [2, 8])
def test_halo_exchange_gloo(world):
    """Partitions, halos (ghost values and ghost rows), batched halo plans and
    [local | ghost] renumbering at 2 and 8 ranks."""
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert dict(out) == {r: 'ok' for r in range(world)}, dict(out)


def test_stable_buckets_is_a_stable_sort_by_owner():
    from paper_2508_17517_b200.dist import stable_buckets
    g = torch.Generator().manual_seed(7)
    for world in (1, 2, 4):
        owner = torch.randint(0, world, (1000,), generator=g)
        perm = stable_buckets(owner, torch.bincount(owner, minlength=world))
        assert torch.equal(perm, torch.argsort(owner, stable=True))
