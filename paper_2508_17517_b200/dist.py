"""Row-strip domain decomposition of the AIRG setup and solve across GPUs
(SURVEY.md 8(e)).  One process per GPU; rank r owns a contiguous block of
global rows at every level (grid strips at level 0, the C points of its fine
strip at the next level, ...), so the global numbering -- and with it every
per-row decision -- is the serial one: a distributed hierarchy is bitwise
the serial hierarchy for the same smoother / coarse polynomials.

Exchanges (torch.distributed over NCCL, all_to_all_single with uneven splits):
  * Halo(part, need): ghost values of the global ids a rank's rows touch;
  * Halo.rows: ghost ROWS (variable length) for the row-local SpGEMMs;
  * allreduce for the DDC histogram / extrema, Luby's undecided count and
    Krylov dot products.
Kernels run on local rows with column ids renumbered in place to
[local | ghost] (the stored order stays the global order, which is what the
bit-exact sums depend on).  Once a level is small (or reaches the truncation
start) it is gathered to every rank and the serial setup continues there,
replicated; the V-cycle does the same below that level.
"""

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .csr import IDX, VAL, SparseMatrix, empty, extract_mapped, take

I64 = torch.int64


class Comm:
    """Collectives on CUDA tensors (NCCL) or CPU tensors (gloo, tests)."""

    def __init__(self, group=None, device=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device or torch.device('cuda', torch.cuda.current_device())

    def a2a(self, send, send_counts, recv_counts):
        out = torch.empty(int(sum(recv_counts)), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(out, send.contiguous(), [int(c) for c in recv_counts],
                               [int(c) for c in send_counts], group=self.group)
        return out

    def allreduce(self, t, op='sum'):
        ops = {'sum': dist.ReduceOp.SUM, 'max': dist.ReduceOp.MAX, 'min': dist.ReduceOp.MIN}
        dist.all_reduce(t, op=ops[op], group=self.group)
        return t

    def sum_int(self, v):
        return int(self.allreduce(torch.tensor([int(v)], dtype=I64, device=self.device)).item())

    def allgather_int(self, v):
        """Per-rank integers (one or a list per rank) -> list over ranks;
        one host read."""
        many = isinstance(v, (list, tuple))
        t = torch.tensor(list(v) if many else [int(v)], dtype=I64, device=self.device)
        out = torch.empty(self.world * t.numel(), dtype=I64, device=self.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        h = out.view(self.world, t.numel()).cpu().tolist()
        return h if many else [x[0] for x in h]

    def sum_dev(self, t):
        """Sum over ranks of a device integer scalar; one host read."""
        return int(self.allreduce(t.reshape(1).to(I64)).item())

    def allgather_dev(self, t):
        """All-gather of a device integer vector -> host list over ranks; one
        host read."""
        t = t.reshape(-1).to(I64)
        out = torch.empty(self.world * t.numel(), dtype=I64, device=t.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.view(self.world, t.numel()).cpu().tolist()

    def allgather_f(self, vals):
        """Per-rank list of floats -> list over ranks; one host read."""
        t = torch.tensor([float(x) for x in vals], dtype=VAL, device=self.device)
        out = torch.empty(self.world * t.numel(), dtype=VAL, device=self.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.view(self.world, t.numel()).cpu().tolist()

    def sum_ints(self, vals):
        """Elementwise sum over ranks of a list of integers; one host read."""
        t = torch.tensor([int(x) for x in vals], dtype=I64, device=self.device)
        return self.allreduce(t).cpu().tolist()

    def allgather_v(self, t):
        """Concatenation over ranks of 1-D tensors of different lengths."""
        counts = self.allgather_int(t.numel())
        m = max(counts) if counts else 0
        pad = torch.zeros(m, dtype=t.dtype, device=t.device)
        pad[:t.numel()] = t
        out = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(out, pad, group=self.group)
        return torch.cat([o[:c] for o, c in zip(out, counts)])


class Part:
    """Contiguous block partition of a global index space."""

    def __init__(self, offsets, device):
        self.off = [int(o) for o in offsets]
        self.n = self.off[-1]
        self.inner = torch.tensor(self.off[1:-1], dtype=I64, device=device)

    @classmethod
    def from_counts(cls, counts, device):
        return cls(np.concatenate([[0], np.cumsum(counts)]).tolist(), device)

    def lo(self, r):
        return self.off[r]

    def hi(self, r):
        return self.off[r + 1]

    def owner(self, g):
        return torch.searchsorted(self.inner, g.to(I64), right=True)


class Halo:
    """Ghost plan: the sorted global ids ``need`` (outside this rank's block)
    and, per peer, which local entries this rank sends."""

    def __init__(self, comm, part, need):
        self.comm, self.part = comm, part
        W, r = comm.world, comm.rank
        self.ghost = need.to(I64)
        self.n_loc = part.hi(r) - part.lo(r)
        self.n = int(self.ghost.numel())
        owners = part.owner(self.ghost) if self.n else torch.zeros(0, dtype=I64, device=comm.device)
        # mat[q][p]: ghosts rank q needs from rank p (one all-gather, one host read)
        mat = comm.allgather_dev(torch.bincount(owners, minlength=W))
        self.recv_counts = mat[r]
        self.send_counts = [mat[q][r] for q in range(W)]
        req = comm.a2a(self.ghost, self.recv_counts, self.send_counts)
        self.send_idx = req - part.lo(r)

    @classmethod
    def many(cls, comm, items):
        """Halo(comm, part, need) for every (part, need) of ``items`` with ONE
        all-gather of the count matrices and ONE all-to-all of the requests
        (instead of two collectives per plan).  Same plans as the per-item
        constructor: ghosts sorted, per-peer requests in ghost order."""
        W, r, K = comm.world, comm.rank, len(items)
        if K == 0:
            return []
        dev = comm.device
        hs, owners = [], []
        for part, need in items:
            h = cls.__new__(cls)
            h.comm, h.part = comm, part
            h.ghost = need.to(I64)
            h.n_loc = part.hi(r) - part.lo(r)
            h.n = int(h.ghost.numel())
            hs.append(h)
            owners.append(part.owner(h.ghost) if h.n else torch.zeros(0, dtype=I64, device=dev))
        counts = torch.stack([torch.bincount(o, minlength=W) for o in owners])  # [K, W]
        mat = np.asarray(comm.allgather_dev(counts)).reshape(W, K, W)  # [q, i, p]
        # send buffer ordered by (peer, item); within one item the ghosts of a
        # peer are contiguous (sorted ids, contiguous partition)
        key = torch.cat([o * K + i for i, o in enumerate(owners)])
        ghosts = torch.cat([h.ghost for h in hs])
        send = ghosts[torch.argsort(key, stable=True)] if ghosts.numel() else ghosts
        send_tot = [int(mat[r, :, p].sum()) for p in range(W)]
        recv_tot = [int(mat[q, :, r].sum()) for q in range(W)]
        req = comm.a2a(send, send_tot, recv_tot)
        # received: peer q, then item i; regroup per item in peer order
        seg = mat[:, :, r]  # [q, i] requests of q for item i
        off = np.concatenate([[0], np.cumsum(seg.reshape(-1))])[:-1].reshape(W, K)
        parts = [np.arange(off[q, i], off[q, i] + seg[q, i]) for i in range(K) for q in range(W)]
        perm = torch.from_numpy(np.concatenate(parts).astype(np.int64)).to(dev) if parts else None
        req = req[perm] if perm is not None and req.numel() else req
        pos = 0
        for i, h in enumerate(hs):
            h.recv_counts = [int(mat[r, i, p]) for p in range(W)]
            h.send_counts = [int(mat[q, i, r]) for q in range(W)]
            ns = int(sum(h.send_counts))
            h.send_idx = req[pos:pos + ns] - h.part.lo(r)
            pos += ns
        return hs

    def values(self, local):
        """Ghost values (in ghost order) of a per-local-row array."""
        return self.comm.a2a(local[self.send_idx], self.send_counts, self.recv_counts)

    def ext(self, local):
        return torch.cat([local, self.values(local)])

    def rows(self, M):
        """Ghost rows of the local-row CSR M (global column ids) -> CSR."""
        dev = M.row_offsets.device
        lens = (M.row_offsets[1:] - M.row_offsets[:-1]).to(I64)
        slen = lens[self.send_idx]
        rlen = self.comm.a2a(slen, self.send_counts, self.recv_counts)
        # element counts per peer (one segmented sum, one host copy)
        def per_peer(counts, lengths):
            seg = torch.repeat_interleave(torch.arange(len(counts), device=dev),
                                          torch.tensor(counts, device=dev),
                                          output_size=int(sum(counts)))
            tot = torch.zeros(len(counts), dtype=I64, device=dev)
            if lengths.numel():
                tot.index_add_(0, seg, lengths)
            return tot
        both = torch.cat([per_peer(self.send_counts, slen), per_peer(self.recv_counts, rlen)])
        both = both.cpu().tolist()
        se, re_ = both[:self.comm.world], both[self.comm.world:]
        starts = M.row_offsets[:-1].to(I64)[self.send_idx]
        tot = int(sum(se))
        if tot:
            first = torch.cumsum(slen, 0) - slen
            idx = (torch.arange(tot, device=dev)
                   - torch.repeat_interleave(first, slen, output_size=tot)
                   + torch.repeat_interleave(starts, slen, output_size=tot))
            scol, sval = M.col_indices[idx], M.values[idx]
        else:
            scol = torch.zeros(0, dtype=IDX, device=dev)
            sval = torch.zeros(0, dtype=VAL, device=dev)
        gcol = self.comm.a2a(scol, se, re_)
        gval = self.comm.a2a(sval, se, re_)
        gptr = torch.zeros(self.n + 1, dtype=I64, device=dev)
        gptr[1:] = torch.cumsum(rlen, 0)
        return gptr.to(IDX), gcol, gval

    def ext_cols(self, col):
        """Global column ids -> ext ids [local | ghost] (order of storage kept)."""
        lo, hi = self.part.lo(self.comm.rank), self.part.hi(self.comm.rank)
        c = col.to(I64)
        loc = (c >= lo) & (c < hi)
        out = torch.where(loc, c - lo, self.n_loc + torch.searchsorted(self.ghost, c))
        return out.to(IDX)


def remote_cols(col, part, rank):
    """Sorted distinct global columns outside this rank's range: a flag per
    global column (one scatter over the column array, one compaction) -- no
    int64 copy of the column array and no sort."""
    lo, hi = part.lo(rank), part.hi(rank)
    f = torch.zeros(part.n, dtype=torch.bool, device=col.device)
    if col.numel():
        f[col] = True
    f[lo:hi] = False
    return f.nonzero().squeeze(1)


def cat_rows(M, gptr, gcol, gval, ncols):
    """Local rows of M followed by ghost rows."""
    nnz = M.nnz
    ptr = torch.cat([M.row_offsets[:-1], gptr + nnz])
    return SparseMatrix(M.nrows + gptr.numel() - 1, ncols, ptr.to(IDX),
                        torch.cat([M.col_indices, gcol]), torch.cat([M.values, gval]))


def with_cols(M, col, ncols):
    return SparseMatrix(M.nrows, ncols, M.row_offsets, col, M.values)


@dataclass
class DMat:
    """Local rows of a row-partitioned global matrix (global column ids)."""

    M: SparseMatrix
    rows: Part
    cols: Part

    def row0(self, rank):
        return self.rows.lo(rank)


@dataclass
class DLevel:
    """One distributed level: operators on local rows (global column ids)."""

    R: SparseMatrix
    A_ff: SparseMatrix
    A_fc: SparseMatrix
    f_loc: torch.Tensor
    c_loc: torch.Tensor
    labels: torch.Tensor
    fine: Part
    fpart: Part
    cpart: Part
    f_smoother: object
    n: int
    n_f: int
    n_c: int
    nnz_A: int
    nnz_R: int
    nnz_Aff: int
    nnz_Afc: int
    ddc_stats: tuple = ()
    pcol: torch.Tensor = None
    halo_R: object = None   # ghost plan of R's columns (fine space), reused by the solve
    halo_F: object = None   # ghost plan of A_ff's columns (F space)


@dataclass
class DHierarchy:
    dlevels: list
    tail: object          # serial Hierarchy of the replicated coarse levels (or None)
    tail_level: int       # global level index where the tail starts
    top: DMat
    comm: Comm
    polys: dict = field(default_factory=dict)
    truncated_at: int = None
    config: object = None
    setup_breakdown: dict = None
    tail_dmat: object = None  # the tail's top level on its row strips (before the gather)

    @property
    def num_levels(self):
        return len(self.dlevels) + (self.tail.num_levels if self.tail else 0)


# ---------------------------------------------------------------------------
# problem generation
# ---------------------------------------------------------------------------

def advection_2d_strips(comm, nx, ny, vx, vy, weights=None):
    """Rank-local grid-row strip of the 2-D upwind operator (problems.py:48-85).
    ``weights`` (per rank) sets relative strip heights; the global numbering,
    and with it every level operator, does not depend on them."""
    r, W = comm.rank, comm.world
    if weights is None:
        rows = [(ny * q) // W * nx for q in range(W + 1)]
    else:
        c = np.concatenate([[0.0], np.cumsum(np.asarray(weights, dtype=np.float64))])
        rows = [int(round(ny * c[q] / c[-1])) * nx for q in range(W + 1)]
    part = Part(rows, comm.device)
    lo, hi = part.lo(r), part.hi(r)
    nnz = L.i64()
    L.call('airg_advection_2d_rows', nx, ny, float(vx), float(vy), lo, hi, None, None, None,
           L.C.byref(nnz), L.stream_handle())
    p, c, v = empty(hi - lo + 1, IDX), empty(nnz.value, IDX), empty(nnz.value, VAL)
    L.call('airg_advection_2d_rows', nx, ny, float(vx), float(vy), lo, hi, L.ptr(p), L.ptr(c),
           L.ptr(v), None, L.stream_handle())
    return DMat(SparseMatrix(hi - lo, part.n, p, c, v), part, part)


def gather_dmat(comm, A):
    """All rows of a distributed matrix on every rank (global SparseMatrix)."""
    M = A.M
    lens = (M.row_offsets[1:] - M.row_offsets[:-1]).to(I64)
    lens_all = comm.allgather_v(lens)
    cols = comm.allgather_v(M.col_indices)
    vals = comm.allgather_v(M.values)
    ptr = torch.zeros(A.rows.n + 1, dtype=I64, device=lens.device)
    ptr[1:] = torch.cumsum(lens_all, 0)
    return SparseMatrix(A.rows.n, A.cols.n, ptr.to(IDX), cols, vals)


# ---------------------------------------------------------------------------
# distributed building blocks
# ---------------------------------------------------------------------------

def _local_index(labels, which):
    return torch.nonzero(labels == which).flatten().to(IDX)


def stable_buckets(owner, counts):
    """Permutation that orders ``owner`` (values 0..k-1, device) by bucket,
    keeping the original order inside each bucket; ``counts`` = bincount
    (device).  Elementwise + cumsum only: no host read."""
    start = torch.cumsum(counts, 0) - counts
    dest = torch.empty_like(owner)
    for q in range(counts.numel()):
        m = owner == q
        dest = torch.where(m, start[q] + torch.cumsum(m.to(I64), 0) - 1, dest)
    perm = torch.empty_like(owner)
    perm[dest] = torch.arange(owner.numel(), device=owner.device, dtype=owner.dtype)
    return perm


def strength_closure(comm, A, theta):
    """Local rows of pattern(S + S^T) (global columns).  ref: splitting.py:86-109

    S^T's local rows come from an all-to-all of the (j, i) pairs by the owner
    of j; the received pairs are ordered by i (rank chunks in rank order,
    each in its sender's row order), so a stable sort by the local row j
    leaves every transposed row sorted.  Host reads: S's size, the
    world x world pair counts."""
    r = comm.rank
    n, lo = A.M.nrows, A.rows.lo(r)
    res = L.C.c_void_p()
    L.call('airg_strength_rows', n, lo, L.ptr(A.M.row_offsets), L.ptr(A.M.col_indices),
           L.ptr(A.M.values), A.M.nnz, float(theta), L.C.byref(res), L.stream_handle())
    S = take(res, values=False)
    dev = S.row_offsets.device
    lens = (S.row_offsets[1:] - S.row_offsets[:-1]).to(I64)
    i_glob = lo + torch.repeat_interleave(torch.arange(n, device=dev, dtype=I64), lens,
                                          output_size=S.nnz)
    j_glob = S.col_indices.to(I64)
    if comm.world > 1:
        owners = A.rows.owner(j_glob)
        cnt = torch.bincount(owners, minlength=comm.world)
        mat = comm.allgather_dev(cnt)
        sc = mat[r]
        rc = [mat[q][r] for q in range(comm.world)]
        perm = stable_buckets(owners, cnt)
        rj = comm.a2a(j_glob[perm], sc, rc)
        ri = comm.a2a(i_glob[perm], sc, rc)
    else:
        rj, ri = j_glob, i_glob
    trow, p2 = torch.sort((rj - lo).to(IDX), stable=True)
    tcol = ri[p2].to(IDX)
    tptr = torch.zeros(n + 1, dtype=I64, device=dev)
    tptr[1:] = torch.cumsum(torch.bincount(trow, minlength=n), 0)
    res = L.C.c_void_p()
    L.call('airg_union_rows', n, L.ptr(S.row_offsets), L.ptr(S.col_indices),
           L.ptr(tptr.to(IDX)), L.ptr(tcol), L.C.byref(res), L.stream_handle())
    return take(res, values=False)


def pmisr(comm, A, clo, seed, max_luby_loops=None):
    """Distributed Luby rounds (splitting.py:127-159); local labels int8."""
    r = comm.rank
    n, lo = A.M.nrows, A.rows.lo(r)
    halo = Halo(comm, A.rows, remote_cols(clo.col_indices, A.rows, r))
    ccol = halo.ext_cols(clo.col_indices)
    w = empty(n, VAL)
    L.call('airg_luby_weights', n, lo, L.ptr(clo.row_offsets), *L.pcg_params(seed), L.ptr(w),
           L.stream_handle())
    w_ext = halo.ext(w)
    dev = w.device
    gid = torch.cat([torch.arange(lo, lo + n, device=dev, dtype=I64), halo.ghost]).to(IDX)
    st = torch.zeros(n + halo.n, dtype=torch.int8, device=dev)
    left = comm.sum_int(n)
    loops = 0
    rem = L.i32()
    # the global undecided count is checked every `every` rounds (a round after
    # convergence changes nothing: no undecided vertex is left to select)
    every = 1 if max_luby_loops is not None else 3
    while left > 0:
        if max_luby_loops is not None and loops >= max_luby_loops:
            break
        if loops > 0 and loops % 120 == 0:
            st[st >= 3] = 1
        mark = 3 + loops % 120
        check = (loops + 1) % every == 0
        L.call('airg_luby_round', n, L.ptr(clo.row_offsets), L.ptr(ccol), L.ptr(w_ext), L.ptr(gid),
               L.ptr(st), mark, 0, None, L.stream_handle())
        st[n:] = halo.values(st[:n])
        L.call('airg_luby_round', n, L.ptr(clo.row_offsets), L.ptr(ccol), L.ptr(w_ext), L.ptr(gid),
               L.ptr(st), mark, 1, L.C.byref(rem) if check else None, L.stream_handle())
        st[n:] = halo.values(st[:n])
        if check:
            left = comm.sum_int(rem.value)
        loops += 1
    labels = empty(n, torch.int8)
    L.call('airg_luby_finish', n, L.ptr(st), L.ptr(labels), L.stream_handle())
    return labels


def ddc_pass(comm, A_ext, labels_ext, n, row0, fraction, nbins, nf, halo):
    """One distributed DDC pass (splitting.py:177-207); labels updated in place
    (ghosts refreshed through ``halo``).  ``nf`` is the global F count before
    the pass; returns (stats, global F count after).  Host reads: the F index
    list, the local ratio extrema, one all-gather of [bad, min, max, sum], the
    histogram, the F count after."""
    from .cfsplit import DDCPassStats
    f_loc = _local_index(labels_ext[:n], 0)
    nf_loc = int(f_loc.numel())
    if nf == 0:
        raise ValueError('zero-size array to reduction operation minimum which has no identity')
    ratio = empty(nf_loc, VAL)
    bad = L.i32()
    mms = np.zeros(3)
    L.call('airg_ddc_ratios', nf_loc, row0, L.ptr(f_loc), L.ptr(A_ext.row_offsets),
           L.ptr(A_ext.col_indices), L.ptr(A_ext.values), L.ptr(labels_ext), L.ptr(ratio),
           L.C.byref(bad), L.hptr(mms), L.stream_handle())
    g = comm.allgather_f([float(bad.value), mms[0], mms[1], mms[2] if nf_loc else 0.0])
    b = int(min(x[0] for x in g))
    if b != 0x7fffffff:
        raise ValueError(f'zero diagonal in fine-fine block (fine row {b}); splitting is not '
                         'usable for reduction')
    lo, hi = min(x[1] for x in g), max(x[2] for x in g)
    sm = 0.0
    for x in g:
        sm += x[3]
    target = fraction * nf
    dev = ratio.device
    if lo == hi:
        allc = abs(nf - target) < target
        cut = lo if allc else hi
        if allc:
            L.call('airg_ddc_convert', nf_loc, L.ptr(f_loc), L.ptr(ratio), cut, 1, L.ptr(labels_ext),
                   None, L.stream_handle())
    else:
        edges = lo + (hi - lo) * np.arange(nbins + 1) / nbins
        edges = np.ascontiguousarray(edges)
        hist = torch.zeros(nbins + 2, dtype=I64, device=dev)
        L.call('airg_ddc_hist', nf_loc, L.ptr(ratio), L.hptr(edges), nbins + 1, L.ptr(hist),
               L.stream_handle())
        hist = comm.allreduce(hist).cpu().numpy()
        above = np.cumsum(hist[::-1])[::-1][1:]          # above[k] = sum_{b > k} hist[b]
        k = nbins - int(np.argmin(np.abs(above - target)[::-1]))
        cut = float(edges[k])
        L.call('airg_ddc_convert', nf_loc, L.ptr(f_loc), L.ptr(ratio), cut, 0, L.ptr(labels_ext),
               None, L.stream_handle())
    labels_ext[n:] = halo.values(labels_ext[:n])
    nf_after = comm.sum_dev((labels_ext[:n] == 0).sum())
    return DDCPassStats(n_f_before=nf, converted=nf - nf_after, ratio_min=lo, ratio_max=hi,
                        ratio_mean=sm / nf, cut=cut), nf_after


def dist_arnoldi_coeffs(comm, A_ff, halo, order, seed):
    """GMRES polynomial (monomial) of a row-strip A_ff (polynomial.py:68-110):
    device SpMV with halo, Gram-Schmidt, lucky-breakdown rule, host
    coefficients from the (identical on every rank) Hessenberg block.  The
    projections of a sweep are formed at once (classical Gram-Schmidt: V^T w,
    one allreduce of j+1 numbers) and both sweeps always run, so the
    recurrence needs no host round trip; the coefficients then differ from the
    reference's modified Gram-Schmidt ones by rounding only, like the serial
    GPU's (whose dot products round differently from the reference)."""
    from .gmres_poly import coeffs_from_hessenberg
    from .csr import spmv
    r = comm.rank
    n, lo, N = A_ff.nrows, halo.part.lo(r), halo.part.n
    m = min(order + 1, N)
    A_ext = with_cols(A_ff, halo.ext_cols(A_ff.col_indices), n + halo.n)
    v = empty(n, VAL)
    L.call('airg_pcg64_fill_at', *L.pcg_params(seed), lo, n, -1.0, 2.0, L.ptr(v), L.stream_handle())

    def allred(t):  # one allreduce, one host read
        return comm.allreduce(t).cpu().numpy()

    b = v / float(np.sqrt(allred(torch.dot(v, v).reshape(1))[0]))
    beta = float(np.sqrt(allred(torch.dot(b, b).reshape(1))[0]))
    if beta == 0:
        raise ValueError('cannot build a Krylov space from a zero vector')
    # The whole recurrence stays on the device (allreduces without host
    # reads): both Gram-Schmidt sweeps always run (the reference's selective
    # second sweep only adds rounding-level corrections when it is skipped),
    # and the lucky breakdown is found afterwards on the host copy of H — the
    # columns after a breakdown are never used.
    dev = v.device
    V = torch.empty((m + 1, n), dtype=VAL, device=dev)
    V[0] = b / beta
    Hd = torch.zeros((m + 1, m), dtype=VAL, device=dev)
    for j in range(m):
        w = spmv(A_ext, halo.ext(V[j]))
        Vj = V[:j + 1]
        h = comm.allreduce(torch.mv(Vj, w))
        w = w - torch.mv(Vj.t(), h)
        h2 = comm.allreduce(torch.mv(Vj, w))
        w = w - torch.mv(Vj.t(), h2)
        hn = torch.sqrt(comm.allreduce(torch.dot(w, w).reshape(1)))
        Hd[:j + 1, j] = h + h2
        Hd[j + 1, j] = hn[0]
        V[j + 1] = w / hn
    H = Hd.cpu().numpy()
    hmax, k = 0.0, m
    for j in range(m):
        hmax = max(hmax, float(np.linalg.norm(H[:j + 2, j])))
        if H[j + 1, j] <= 1e-14 * hmax:
            H[j + 1, j] = 0.0
            k = j + 1
            break
    if np.max(np.abs(H[:k + 1, :k])) == 0.0:
        raise ValueError('matrix is numerically zero on the Krylov space')
    return coeffs_from_hessenberg(H[:k + 1, :k].copy(), k, beta, order)


def _spgemm(A, B, ncols, negate=False, mode=0, tol=0.0, lump=False, row0=0):
    res = L.C.c_void_p()
    L.call('airg_spgemm_ex', A.nrows, B.nrows, ncols, L.ptr(A.row_offsets), L.ptr(A.col_indices),
           L.ptr(A.values), L.ptr(B.row_offsets), L.ptr(B.col_indices), L.ptr(B.values),
           1 if negate else 0, mode, float(tol), 1 if lump else 0, int(row0), L.C.byref(res),
           L.stream_handle())
    out = take(res)
    return SparseMatrix(out.nrows, ncols, out.row_offsets, out.col_indices, out.values)


# ---------------------------------------------------------------------------
# distributed setup
# ---------------------------------------------------------------------------

class _Ticker:
    """Phase timer for the distributed setup: each call charges the stream
    time since the previous call to the named phase.  CUDA events in stream
    order (the interval includes any device idle time waiting for the host);
    the elapsed times are summed once, at tick(None), instead of
    synchronising the device at every phase boundary."""

    def __init__(self, sink):
        import os
        self.sink = sink
        self.per_level = bool(os.environ.get('AIRG_DIST_LEVEL_TIMES'))
        self.level = 0
        self.pending = []
        self.prev = torch.cuda.Event(enable_timing=True)
        self.prev.record()

    def __call__(self, phase):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        if phase is not None:
            self.pending.append((phase, self.level, self.prev, e))
        self.prev = e
        if phase is None:
            self.flush()

    def flush(self):
        if self.pending:
            self.pending[-1][3].synchronize()
        for phase, level, e0, e1 in self.pending:
            dt = e0.elapsed_time(e1) / 1e3
            self.sink[phase] = self.sink.get(phase, 0.0) + dt
            if self.per_level:
                key = f'{phase}@{level}'
                self.sink[key] = self.sink.get(key, 0.0) + dt
        self.pending = []

    def note(self, key, value):
        if self.per_level:
            self.sink[f'{key}@{self.level}'] = value


def setup_distributed(comm, A, cfg, poly_inject=None, replicate_below=None, force=False):
    """AIRG setup (hierarchy.py:365-448) on a row-partitioned matrix.  Levels
    with more than ``replicate_below`` rows (and below the truncation start)
    are built distributed; the rest is built on every rank from the gathered
    level matrix with the serial code.  ``force`` runs the distributed levels
    even on a single rank (overhead measurements)."""
    from .amg_setup import (SETUP_PHASES, SEED_SMOOTHER, SEED_SPLIT, build_levels, derive_seed,
                            resolve_truncate_start, finalize_complexities, Hierarchy)
    cfg.validate()
    if replicate_below is None:
        import os
        replicate_below = int(os.environ.get('AIRG_REPLICATE_BELOW', 20000))
    if cfg.inverse_type != 'arnoldi' or cfg.r_drop != 0:
        raise ValueError('the distributed setup supports inverse_type="arnoldi" with r_drop=0')
    inj = poly_inject or {}
    polys = {}
    timings = {p: 0.0 for p in SETUP_PHASES}
    r = comm.rank
    truncate_start = resolve_truncate_start(cfg, A.rows.n)
    tick = _Ticker(timings)
    dlevels = []
    level = 0
    cur = A
    while (cur.rows.n > replicate_below and (comm.world > 1 or force) and level < cfg.max_levels
           and cur.rows.n > cfg.min_coarse_size
           and not (cfg.auto_truncate_tol is not None and level >= truncate_start)):
        n, lo = cur.M.nrows, cur.rows.lo(r)
        dev = cur.M.values.device
        # ---- CF splitting ----
        clo = strength_closure(comm, cur, cfg.strong_threshold)
        tick('cf_split.strength')
        labels = pmisr(comm, cur, clo, derive_seed(cfg.seed, level, SEED_SPLIT))
        tick('cf_split.pmisr')
        halo_a = Halo(comm, cur.rows, remote_cols(cur.M.col_indices, cur.rows, r))
        A_ext = with_cols(cur.M, halo_a.ext_cols(cur.M.col_indices), n + halo_a.n)
        lab_ext = halo_a.ext(labels)
        tick('cf_split.halo')
        stats = []
        nf_glob = comm.sum_dev((lab_ext[:n] == 0).sum())
        for _ in range(cfg.ddc_its):
            if nf_glob == 0:
                break
            st_, nf_glob = ddc_pass(comm, A_ext, lab_ext, n, lo, cfg.ddc_fraction, cfg.ddc_bins,
                                    nf_glob, halo_a)
            stats.append(st_)
        nc_glob = cur.rows.n - nf_glob
        tick('cf_split.ddc')
        if nc_glob == cur.rows.n:
            raise ValueError(f'splitting produced no F points at level {level}')
        if nc_glob > 0:
            ch = L.i32()
            L.call('airg_repair_split', n, L.ptr(A_ext.row_offsets), L.ptr(A_ext.col_indices),
                   L.ptr(lab_ext), L.C.byref(ch), L.stream_handle())
            lab_ext[n:] = halo_a.values(lab_ext[:n])
        labels = lab_ext[:n].clone()
        f_loc, c_loc = _local_index(labels, 0), _local_index(labels, 1)
        fc_all = comm.allgather_int([f_loc.numel(), c_loc.numel()])
        nf_all = [x[0] for x in fc_all]
        nc_all = [x[1] for x in fc_all]
        if sum(nc_all) == 0 or sum(nf_all) == 0:
            break  # the replicated tail builds the coarse solver here
        fpart, cpart = Part.from_counts(nf_all, dev), Part.from_counts(nc_all, dev)
        fpos0, cpos0 = fpart.lo(r), cpart.lo(r)
        gpos = torch.zeros(n, dtype=IDX, device=dev)
        gpos[f_loc.long()] = torch.arange(fpos0, fpos0 + f_loc.numel(), device=dev, dtype=IDX)
        gpos[c_loc.long()] = torch.arange(cpos0, cpos0 + c_loc.numel(), device=dev, dtype=IDX)
        gpos_ext = halo_a.ext(gpos)
        fmap, cmap = empty(n + halo_a.n, IDX), empty(n + halo_a.n, IDX)
        L.call('airg_label_colmap', n + halo_a.n, L.ptr(lab_ext), 0, L.ptr(gpos_ext), L.ptr(fmap),
               L.stream_handle())
        L.call('airg_label_colmap', n + halo_a.n, L.ptr(lab_ext), 1, L.ptr(gpos_ext), L.ptr(cmap),
               L.stream_handle())
        A_ff = extract_mapped(A_ext, f_loc, fmap, fpart.n)
        A_fc = extract_mapped(A_ext, f_loc, cmap, cpart.n)
        A_cf = extract_mapped(A_ext, c_loc, fmap, fpart.n)
        tick('extract')
        # ---- smoother ----
        halo_ff = Halo(comm, fpart, remote_cols(A_ff.col_indices, fpart, r))
        sm = inj.get(('smoother', level))
        if sm is None:
            sm = dist_arnoldi_coeffs(comm, A_ff, halo_ff, cfg.poly_order,
                                     derive_seed(cfg.seed, level, SEED_SMOOTHER))
        polys[('smoother', level)] = sm
        # ---- fixed-sparsity assembly on local rows with ghost rows of A_ff ----
        gp, gc, gv = halo_ff.rows(A_ff)
        Aff_rows = cat_rows(A_ff, gp, gc, gv, fpart.n)
        rowmap = torch.full((fpart.n,), -1, dtype=IDX, device=dev)
        rowmap[fpos0:fpos0 + A_ff.nrows] = torch.arange(A_ff.nrows, device=dev, dtype=IDX)
        if halo_ff.n:
            rowmap[halo_ff.ghost] = torch.arange(A_ff.nrows, A_ff.nrows + halo_ff.n, device=dev,
                                                 dtype=IDX)
        coef = np.ascontiguousarray(sm.coeffs, dtype=np.float64)
        res = L.C.c_void_p()
        L.call('airg_poly_assemble_ex', A_ff.nrows, fpos0, L.ptr(Aff_rows.row_offsets),
               L.ptr(Aff_rows.col_indices), L.ptr(Aff_rows.values), L.ptr(rowmap), len(coef),
               L.hptr(coef), L.ptr(A_ff.row_offsets), L.ptr(A_ff.col_indices), L.C.byref(res),
               L.stream_handle())
        Ahat = take(res)
        Ahat = SparseMatrix(Ahat.nrows, fpart.n, Ahat.row_offsets, Ahat.col_indices, Ahat.values)
        tick('polynomial')
        # ---- Z = -A_cf Ahat ----
        halo_z = Halo(comm, fpart, remote_cols(A_cf.col_indices, fpart, r))
        tick('spgemm_R.halo')
        Ahat_rows = cat_rows(Ahat, *halo_z.rows(Ahat), fpart.n)
        tick('spgemm_R.rows')
        Z = _spgemm(with_cols(A_cf, halo_z.ext_cols(A_cf.col_indices), Ahat_rows.nrows), Ahat_rows,
                    fpart.n, negate=True)
        tick('spgemm_R.Z')
        # ---- R = [Z I] in the fine numbering ----
        halo_zc = Halo(comm, fpart, remote_cols(Z.col_indices, fpart, r))
        fine_of_f = (lo + f_loc.long()).to(IDX)
        f_ext = halo_zc.ext(fine_of_f)
        Zx = with_cols(Z, halo_zc.ext_cols(Z.col_indices), f_loc.numel() + halo_zc.n)
        res = L.C.c_void_p()
        L.call('airg_restriction', cur.rows.n, Zx.nrows, L.ptr(Zx.row_offsets), L.ptr(Zx.col_indices),
               L.ptr(Zx.values), L.ptr(f_ext), L.ptr((lo + c_loc.long()).to(IDX)), L.C.byref(res),
               L.stream_handle())
        R = take(res)
        tick('spgemm_R')
        # ---- one-point P, A P, R (A P) with drop/lump ----
        pcol = empty(n, IDX)
        L.call('airg_prolong_onepoint', n, L.ptr(A_ext.row_offsets), L.ptr(A_ext.col_indices),
               L.ptr(A_ext.values), L.ptr(lab_ext), L.ptr(gpos_ext), L.ptr(pcol), L.stream_handle())
        pcol_ext = halo_a.ext(pcol)
        res = L.C.c_void_p()
        L.call('airg_ap_onepoint', A_ext.nrows, A_ext.ncols, cpart.n, L.ptr(A_ext.row_offsets),
               L.ptr(A_ext.col_indices), L.ptr(A_ext.values), L.ptr(pcol_ext), L.C.byref(res),
               L.stream_handle())
        AP = take(res)
        AP = SparseMatrix(AP.nrows, cpart.n, AP.row_offsets, AP.col_indices, AP.values)
        tick('prolongator')
        halo_r = Halo(comm, cur.rows, remote_cols(R.col_indices, cur.rows, r))
        tick('spgemm_coarse.halo')
        AP_rows = cat_rows(AP, *halo_r.rows(AP), cpart.n)
        tick('spgemm_coarse.rows')
        Rx = with_cols(R, halo_r.ext_cols(R.col_indices), AP_rows.nrows)
        if cfg.a_drop > 0:
            Ac = _spgemm(Rx, AP_rows, cpart.n, mode=1, tol=cfg.a_drop, lump=cfg.lump, row0=cpos0)
        else:
            Ac = _spgemm(Rx, AP_rows, cpart.n)
        tick('spgemm_coarse.RAP')
        tick.note('nnz_R', R.nnz)
        tick.note('nnz_AP', AP_rows.nnz)
        tick.note('nnz_Ac', Ac.nnz)
        tick.note('n', n)
        nnz_A, nnz_R, nnz_Aff, nnz_Afc = comm.sum_ints([cur.M.nnz, R.nnz, A_ff.nnz, A_fc.nnz])
        dlevels.append(DLevel(R=R, A_ff=A_ff, A_fc=A_fc, f_loc=f_loc, c_loc=c_loc, labels=labels,
                              fine=cur.rows, fpart=fpart, cpart=cpart, f_smoother=sm,
                              n=cur.rows.n, n_f=fpart.n, n_c=cpart.n,
                              nnz_A=nnz_A, nnz_R=nnz_R, nnz_Aff=nnz_Aff, nnz_Afc=nnz_Afc,
                              ddc_stats=tuple(stats), pcol=pcol, halo_R=halo_r, halo_F=halo_ff))
        tick('spgemm_coarse')
        cur = DMat(Ac, cpart, cpart)
        level += 1
        tick.level = level
    # ---- replicated tail ----
    full = gather_dmat(comm, cur)
    tick('gather_tail')
    levels, coarsest, solver, trunc = build_levels(full, cfg, level, truncate_start, inj, polys,
                                                   timings)
    timings.pop('_per_level', None)
    tail = Hierarchy(levels=levels, coarsest_A=coarsest, coarse_solver=solver, top_A=full,
                     truncated_at=trunc, config=cfg, setup_breakdown=timings)
    tail.polys = polys
    finalize_complexities(tail)
    tick(None)
    return DHierarchy(dlevels=dlevels, tail=tail, tail_level=level, top=A, comm=comm, polys=polys,
                      truncated_at=trunc, config=cfg, setup_breakdown=timings, tail_dmat=cur)


# ---------------------------------------------------------------------------
# distributed solve (solve.py:95-167): V-cycle on row strips with halos;
# below the distributed levels the replicated tail runs the serial plan.
# ---------------------------------------------------------------------------

_NATIVE_COMMS = {}


def native_comm(comm):
    """The process's NCCL communicator for the native plans (created once)."""
    key = (comm.rank, comm.world, id(comm.group))
    if key not in _NATIVE_COMMS:
        uid = torch.zeros(128, dtype=torch.uint8, device=comm.device)
        if comm.rank == 0:
            buf = L.C.create_string_buffer(128)
            L.call('airg_nccl_unique_id', buf)
            uid.copy_(torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8))
        dist.broadcast(uid, 0, group=comm.group)
        h = L.C.c_void_p()
        L.call('airg_comm_create', bytes(uid.cpu().numpy().tobytes()), comm.rank, comm.world,
               L.C.byref(h))
        _NATIVE_COMMS[key] = h
    return _NATIVE_COMMS[key]


class DistSolver:
    def __init__(self, H):
        self.H = H
        comm = H.comm
        r = comm.rank
        self.comm = comm
        self.lv = []
        top = H.top
        # every ghost plan the setup did not leave behind, built in one batch
        # (one all-gather + one all-to-all): the R and A_ff plans of the setup
        # are the solve's; A_fc and the top operator need new ones
        want = []
        for d in H.dlevels:
            if d.halo_R is None:
                want.append((d.fine, remote_cols(d.R.col_indices, d.fine, r)))
            want.append((d.cpart, remote_cols(d.A_fc.col_indices, d.cpart, r)))
            if d.halo_F is None:
                want.append((d.fpart, remote_cols(d.A_ff.col_indices, d.fpart, r)))
        want.append((top.rows, remote_cols(top.M.col_indices, top.rows, r)))
        built = iter(Halo.many(comm, want))
        for d in H.dlevels:
            hR = d.halo_R if d.halo_R is not None else next(built)
            hC = next(built)
            hF = d.halo_F if d.halo_F is not None else next(built)
            self.lv.append(dict(
                R=with_cols(d.R, hR.ext_cols(d.R.col_indices), hR.n_loc + hR.n),
                hR=hR,
                Afc=with_cols(d.A_fc, hC.ext_cols(d.A_fc.col_indices), hC.n_loc + hC.n), hC=hC,
                Aff=with_cols(d.A_ff, hF.ext_cols(d.A_ff.col_indices), hF.n_loc + hF.n), hF=hF,
                f=d.f_loc.long(), c=d.c_loc.long(), n=d.fine.hi(r) - d.fine.lo(r),
                coef=np.asarray(d.f_smoother.coeffs, dtype=np.float64)))
        self.htop = next(built)
        self.Atop = with_cols(top.M, self.htop.ext_cols(top.M.col_indices),
                              self.htop.n_loc + self.htop.n)
        # partition of the first replicated level (the tail's top matrix)
        if H.dlevels:
            self.tail_part = H.dlevels[-1].cpart
        else:
            self.tail_part = top.rows

    def _smooth(self, L_, rhs):
        from .csr import spmv
        c = L_['coef']
        d = len(c) - 1
        y = c[d] * rhs
        for j in range(d - 1, -1, -1):
            y = spmv(L_['Aff'], L_['hF'].ext(y)) + c[j] * rhs
        return y

    def vcycle(self, lev, r_loc):
        from .amg_solve import SolveConfig, vcycle as serial_vcycle
        from .csr import spmv
        comm = self.comm
        if lev == len(self.lv):
            r_full = comm.allgather_v(r_loc)
            e_full = serial_vcycle(self.H.tail, 0, r_full, SolveConfig())
            p = self.tail_part
            return e_full[p.lo(comm.rank):p.hi(comm.rank)]
        L_ = self.lv[lev]
        rc = spmv(L_['R'], L_['hR'].ext(r_loc))
        ec = self.vcycle(lev + 1, rc)
        rhs = r_loc[L_['f']] - spmv(L_['Afc'], L_['hC'].ext(ec))
        ef = self._smooth(L_, rhs)
        e = torch.zeros(L_['n'], dtype=VAL, device=r_loc.device)
        e[L_['f']] = ef
        e[L_['c']] = ec
        return e

    def norm(self, v):
        return float(np.sqrt(self.comm.allreduce(torch.dot(v, v).reshape(1)).item()))

    # ---- native plan: C++ V-cycle with NCCL halos, graph-captured -------------
    def _native(self):
        if getattr(self, '_dplan', None) is not None:
            return self._dplan
        from .amg_solve import _pool
        comm = self.comm
        h = L.C.c_void_p()
        L.call('airg_dplan_create', native_comm(comm), len(self.lv), L.C.byref(h))
        keep = []

        def set_halo(level, which, halo):
            si = halo.send_idx.to(IDX).contiguous()
            sc = np.ascontiguousarray(halo.send_counts, dtype=np.int32)
            rc = np.ascontiguousarray(halo.recv_counts, dtype=np.int32)
            keep.extend([si, sc, rc])
            L.call('airg_dplan_set_halo', h, level, which, halo.n_loc, si.numel(), L.ptr(si),
                   L.hptr(sc), L.hptr(rc))

        for l, Lv in enumerate(self.lv):
            set_halo(l, 0, Lv['hR'])
            set_halo(l, 1, Lv['hC'])
            set_halo(l, 2, Lv['hF'])
            f32, c32 = Lv['f'].to(IDX).contiguous(), Lv['c'].to(IDX).contiguous()
            coef = np.ascontiguousarray(Lv['coef'])
            keep.extend([f32, c32, coef])
            R, Fc, Ff = Lv['R'], Lv['Afc'], Lv['Aff']
            L.call('airg_dplan_set_level', h, l, Lv['n'], int(f32.numel()), int(c32.numel()),
                   L.ptr(R.row_offsets), L.ptr(R.col_indices), L.ptr(R.values), R.nnz,
                   L.ptr(Fc.row_offsets), L.ptr(Fc.col_indices), L.ptr(Fc.values), Fc.nnz,
                   L.ptr(Ff.row_offsets), L.ptr(Ff.col_indices), L.ptr(Ff.values), Ff.nnz,
                   L.ptr(f32), L.ptr(c32), len(coef), L.hptr(coef))
        set_halo(0, 3, self.htop)
        self._set_dist_coarse(h, keep)
        T = self.Atop
        L.call('airg_dplan_set_top', h, T.nrows, L.ptr(T.row_offsets), L.ptr(T.col_indices),
               L.ptr(T.values), T.nnz)
        # a plan of the tail's pool dedicated to this distributed plan (never released)
        tail = _pool(self.H.tail).acquire(self.H.tail, False)
        p = self.tail_part
        counts = np.ascontiguousarray(np.diff(p.off), dtype=np.int32)
        L.call('airg_dplan_finish', h, tail.h, L.hptr(counts))
        self._keep = keep
        self._dplan = h
        return h

    def _set_dist_coarse(self, h, keep):
        """configs[3]: when the tail is the coarsest grid alone (the hierarchy
        was truncated at the first replicated level) and its solver is the
        Newton polynomial, apply it on the row strips of the coarsest
        operator instead of gathering the grid to every rank
        (AIRG_DIST_COARSE=0 keeps the replicated solve)."""
        import os
        from .gmres_poly import newton_units
        H, comm = self.H, self.comm
        T = H.tail
        if (comm.world == 1 or T is None or T.num_levels != 0 or H.tail_dmat is None
                or T.coarse_solver.kind != 'newton_roots'
                or os.environ.get('AIRG_DIST_COARSE', '1') == '0'):
            return
        Cd = H.tail_dmat
        r = comm.rank
        halo = Halo(comm, Cd.rows, remote_cols(Cd.M.col_indices, Cd.rows, r))
        Cx = with_cols(Cd.M, halo.ext_cols(Cd.M.col_indices), halo.n_loc + halo.n)
        si = halo.send_idx.to(IDX).contiguous()
        sc = np.ascontiguousarray(halo.send_counts, dtype=np.int32)
        rc = np.ascontiguousarray(halo.recv_counts, dtype=np.int32)
        t, a1, a2 = newton_units(T.coarse_solver.roots)
        keep.extend([Cx, si, sc, rc, t, a1, a2])
        L.call('airg_dplan_set_dcoarse', h, Cx.nrows, L.ptr(Cx.row_offsets), L.ptr(Cx.col_indices),
               L.ptr(Cx.values), Cx.nnz, si.numel(), L.ptr(si), L.hptr(sc), L.hptr(rc), len(t),
               L.hptr(t), L.hptr(a1), L.hptr(a2))
        self.dist_coarse = True

    def __del__(self):
        try:
            if getattr(self, '_dplan', None) is not None:
                L.load().airg_dplan_destroy(self._dplan)
        except Exception:
            pass

    def solve(self, b, x0, cfg):
        """Native distributed Richardson (every iteration one captured graph
        with NCCL halo exchanges); b, x0 local device vectors."""
        import ctypes as C
        from .amg_solve import DivergenceError, SolveStats
        cfg.validate()
        if cfg.f_smooth_its != 1:
            raise ValueError('the distributed solve supports f_smooth_its=1')
        h = self._native()
        x = x0.clone()
        hist = np.zeros(cfg.max_iters + 1)
        its, conv = C.c_int(0), C.c_int(0)
        st = L.load().airg_dplan_richardson(h, L.ptr(b), L.ptr(x), cfg.rtol, cfg.atol,
                                            cfg.max_iters, L.hptr(hist), C.byref(its),
                                            C.byref(conv), L.stream_handle())
        if st == L.ERR_DIVERGED:
            raise DivergenceError(L.last_error(), its.value)
        L.check(st, 'airg_dplan_richardson')
        return x, SolveStats(iterations=its.value, residual_history=list(hist[:its.value + 1]),
                             converged=bool(conv.value), cycle_complexity=0.0,
                             storage_complexity=0.0, flops_per_cycle=0)

    def richardson(self, b, x0, cfg):
        """Richardson preconditioned by the distributed V-cycle; b, x0 local."""
        from .amg_solve import DivergenceError, SolveStats
        from .csr import spmv
        cfg.validate()
        x = x0.clone()
        r = b - spmv(self.Atop, self.htop.ext(x))
        rn = self.norm(r)
        hist = [rn]
        bn = self.norm(b)
        thr = max(cfg.rtol * (bn if bn > 0 else rn), cfg.atol)
        conv, its = rn <= thr, 0
        while not conv and its < cfg.max_iters:
            x = x + self.vcycle(0, r)
            r = b - spmv(self.Atop, self.htop.ext(x))
            rn = self.norm(r)
            its += 1
            hist.append(rn)
            if not np.isfinite(rn):
                raise DivergenceError(f'non-finite residual at iteration {its}', its)
            if rn > 1e8 * hist[0]:
                raise DivergenceError(f'residual grew by more than 1e+08 at iteration {its}', its)
            conv = rn <= thr
        return x, SolveStats(iterations=its, residual_history=hist, converged=conv,
                             cycle_complexity=0.0, storage_complexity=0.0, flops_per_cycle=0)


def dist_cycle_bytes(S, include_top=True):
    """Algorithmic HBM bytes one rank moves per distributed Richardson
    iteration (same accounting as amg_solve.count_cycle_bytes): its local rows
    of every distributed level, the whole replicated tail, and the top
    residual on its strip.  Halo payloads are not HBM traffic of the
    kernels' operands and are left out."""
    from .amg_solve import _spmat_bytes, count_cycle_bytes
    tot = 0
    for Lv in S.lv:
        nf, nc, n = int(Lv['f'].numel()), int(Lv['c'].numel()), Lv['n']
        d = len(Lv['coef']) - 1
        tot += _spmat_bytes(Lv['R']) + 8 * n + 8 * nc
        tot += _spmat_bytes(Lv['Afc']) + 8 * nc + 16 * nf
        tot += 16 * nf + d * (_spmat_bytes(Lv['Aff']) + 24 * nf)
        tot += 16 * n
    if getattr(S, 'dist_coarse', False):
        # the Newton units on this rank's strip of the coarsest operator: per
        # unit the SpMV(s) plus x, u, w (z) read and x, u, x0, u0 written
        from .gmres_poly import newton_units
        C = S.H.tail_dmat.M
        t, _, _ = newton_units(S.H.tail.coarse_solver.roots)
        spm = _spmat_bytes(C)
        for ty in t:
            tot += (2 * spm + 72 * C.nrows) if ty else (spm + 56 * C.nrows)
    else:
        tot += count_cycle_bytes(S.H.tail, include_top=False)
    if include_top:
        tot += _spmat_bytes(S.Atop) + 40 * S.Atop.nrows
    return int(tot)
