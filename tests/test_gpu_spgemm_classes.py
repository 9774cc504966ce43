"""Bitwise parity of every SpGEMM row class against the oracle (scipy
csr_matmat semantics, sparse.py:222-240) -- plain products and the fused
drop/lump epilogue (sparse.py:307-352) of the Galerkin product.

The library routes each output row by its column window and length:
  both:    registers (<= 8 / <= 16 products and A entries: the row merged
           with shuffles, 8 / 16 lanes per row);
  count:   hash set (<= 64 products), span bitmap (window <= 4096 / <= 16384 /
           <= 65536 columns), hash set (<= 512 products), CTA hash set (longer),
           global tables (overflow);
  numeric: span path by output length (<= 256 ... <= 4096), hash warp per
           row (<= 32, <= 128), CTA per row (<= 512 ... <= 8192), global
           tables (> 8192).
The synthetic rows below are built so every one of these classes receives
rows: each A row owns private B rows whose columns are drawn from a pool of
about L columns inside a window of W columns (W <= 65536 -> span path,
W > 65536 -> hash path), values from a small set so that sums cancel exactly
(structural zeros) and magnitudes from 1e-12 to 1 so that the drop rule
fires."""

import ctypes as C
import zlib

import numpy as np
import pytest

from oracle import airg_oracle as O
from tests.gpu_util import dev_csr, host_csr

pytestmark = pytest.mark.gpu


def _case(rng, nrows, L, W, ka, bl, ncols, cancel=True):
    """A (nrows x K) with ka entries per row; B (K x ncols) with bl entries
    per row drawn from a per-A-row pool of L columns in a window of W."""
    K = nrows * ka
    ar, ac = np.repeat(np.arange(nrows), ka), np.arange(K)
    br, bc = [], []
    base = rng.integers(0, max(1, ncols - W), size=nrows)
    for i in range(nrows):
        pool = np.sort(rng.choice(W, size=min(L, W), replace=False)) + base[i]
        if i % 3 == 0 and base[i] <= i < base[i] + W:   # diagonal in the pool for some rows
            pool[0] = i
        for j in range(ka):
            br.append(np.full(min(bl, len(pool)), i * ka + j))
            bc.append(np.sort(rng.choice(pool, size=min(bl, len(pool)), replace=False)))
    br, bc = np.concatenate(br), np.concatenate(bc)
    if cancel:
        av = rng.choice([1.0, -1.0, 0.5, -2.0], size=K)
        bv = rng.choice([1.0, -1.0, 0.25, 3.0, 0.0], size=len(br))
        # a spread of magnitudes so that a relative drop tolerance fires
        bv *= 10.0 ** rng.integers(-12, 1, size=len(br))
    else:
        av = rng.standard_normal(K)
        bv = rng.standard_normal(len(br))
    A = O.from_triplets(nrows, K, ar, ac, av)
    B = O.from_triplets(K, ncols, br, bc, bv)
    return A, B


def same(M_dev, M_or):
    H = host_csr(M_dev)
    assert (H.nrows, H.ncols) == (M_or.nrows, M_or.ncols)
    assert np.array_equal(H.ptr, M_or.ptr)
    assert np.array_equal(H.col, M_or.col)
    assert H.val.tobytes() == M_or.val.tobytes()


def _spgemm_ex(A, B, mode, tol, lump, negate=False):
    from paper_2508_17517_b200 import _lib as L
    from paper_2508_17517_b200.csr import take
    Ad, Bd = dev_csr(A), dev_csr(B)
    res = C.c_void_p()
    L.call('airg_spgemm_ex', A.nrows, A.ncols, B.ncols, L.ptr(Ad.row_offsets),
           L.ptr(Ad.col_indices), L.ptr(Ad.values), L.ptr(Bd.row_offsets), L.ptr(Bd.col_indices),
           L.ptr(Bd.values), 1 if negate else 0, mode, float(tol), 1 if lump else 0, 0,
           C.byref(res), L.stream_handle())
    return take(res)


def _drop_lump_rows(M, tol, lump):
    """Oracle drop/lump of the first M.nrows rows of the square extension."""
    n = M.ncols
    ptr = np.concatenate([M.ptr, np.full(n - M.nrows, M.ptr[-1])])
    Sq = O._mk(n, n, ptr, M.col, M.val)
    D = O.drop_lump(Sq, tol, lump)
    m = M.nrows
    return O._mk(m, n, D.ptr[:m + 1], D.col[:D.ptr[m]], D.val[:D.ptr[m]])


# (label, rows, L, W, ka, bl): output length ~L, window W
CASES = [
    ('reg<=8', 400, 8, 40, 2, 3),          # <= 8 products: register class, 8 lanes per row
    ('reg<=16', 300, 14, 60, 4, 4),        # <= 16 products: register class, 16 lanes
    ('hash<=32', 300, 24, 200, 6, 8),
    ('hash<=128', 200, 100, 600, 8, 8),
    ('hash512cnt', 100, 300, 90000, 4, 100),
    ('span<=256', 120, 200, 3000, 12, 60),
    ('span<=512', 80, 450, 4000, 10, 120),
    ('span<=1024', 48, 900, 12000, 12, 200),
    ('span<=2048', 24, 1800, 15000, 12, 400),
    ('span<=4096', 8, 3600, 16000, 10, 900),
    ('span64k<=1024', 24, 900, 40000, 10, 220),
    ('span64k<=4096', 6, 3500, 60000, 10, 900),
    ('hashblk<=512', 40, 400, 90000, 8, 120),
    ('hashblk<=1024', 24, 900, 90000, 10, 220),
    ('hashblk<=2048', 12, 1800, 90000, 10, 450),
    ('hashblk<=4096', 6, 3500, 90000, 10, 900),
    ('span>4096->hash<=8192', 4, 7000, 16000, 10, 1800),
    ('hash>8192->global', 2, 12000, 100000, 10, 3000),
]


@pytest.mark.parametrize('label,nrows,L,W,ka,bl', CASES, ids=[c[0] for c in CASES])
def test_spgemm_class_bitwise(label, nrows, L, W, ka, bl):
    import paper_2508_17517_b200 as G
    rng = np.random.default_rng(zlib.crc32(label.encode()))
    ncols = max(W + 2 * nrows + 10, 2 * nrows)
    A, B = _case(rng, nrows, L, W, ka, bl, ncols)
    want = O.spgemm(A, B)
    assert np.any(want.val == 0.0)   # exact cancellations / structural zeros exercised
    same(G.spgemm(dev_csr(A), dev_csr(B)), want)
    neg = O._mk(want.nrows, want.ncols, want.ptr, want.col, -want.val)
    same(G.spgemm(dev_csr(A), dev_csr(B), negate=True), neg)
    for tol, lump in ((1e-6, True), (1e-3, True), (1e-6, False)):
        same(_spgemm_ex(A, B, 1, tol, lump), _drop_lump_rows(want, tol, lump))


def test_spgemm_mixed_classes_one_call():
    """All classes in ONE product (concurrent class launches on forked
    streams write disjoint rows of the same output)."""
    import paper_2508_17517_b200 as G
    rng = np.random.default_rng(11)
    parts = [_case(rng, n // 4 + 1, L, W, ka, bl, 110000, cancel=(i % 2 == 0))
             for i, (_, n, L, W, ka, bl) in enumerate(CASES[:-1])]
    import scipy.sparse as sps
    A = O.from_scipy(sps.block_diag([p[0].sp() for p in parts], format='csr'))
    B = O.from_scipy(sps.vstack([p[1].sp() for p in parts], format='csr'))
    want = O.spgemm(A, B)
    same(G.spgemm(dev_csr(A), dev_csr(B)), want)
    same(_spgemm_ex(A, B, 1, 1e-6, True), _drop_lump_rows(want, 1e-6, True))
