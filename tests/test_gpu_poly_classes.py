"""Bitwise parity of every masked-polynomial-assembly row class against the
oracle (polynomial.py:372-416 / sparse.py:243-263).

The library classes each pattern row by length (all powers in registers,
8 / 16 lanes per row, for rows of <= 8 / <= 16 entries; warp per row below 512
entries -- its A rows held 1/2/4/8 x 32 entries per lane in the pipeline --,
CTA per row from 512, CTA with a global-memory working set when it exceeds
shared memory) and by column window (bitmap position map for windows
<= 8192 columns, hash table beyond).  The matrices below have short local rows
plus "hub" rows of chosen lengths in narrow or wide windows, so every class
receives rows."""

import numpy as np
import pytest

from oracle import airg_oracle as O
from tests.gpu_util import dev_csr, dev_poly, host_csr

pytestmark = pytest.mark.gpu


def same(M_dev, M_or):
    H = host_csr(M_dev)
    assert (H.nrows, H.ncols) == (M_or.nrows, M_or.ncols)
    assert np.array_equal(H.ptr, M_or.ptr)
    assert np.array_equal(H.col, M_or.col)
    assert H.val.tobytes() == M_or.val.tobytes()


def hub_matrix(seed, n, hubs):
    """n x n: each row ~6 entries within +-40 of the diagonal; hub rows
    (row, length, window) draw `length` columns from a window of `window`
    columns around the row (clipped to [0, n))."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        c = np.unique(np.clip(i + rng.integers(-40, 41, size=6), 0, n - 1))
        rows.append(np.full(len(c), i))
        cols.append(c)
    for r, length, window in hubs:
        lo = max(0, min(r - window // 2, n - window))
        c = np.unique(lo + rng.choice(window, size=length, replace=False))
        rows.append(np.full(len(c), r))
        cols.append(c)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    key = np.unique(rows * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(len(rows)) / np.sqrt(np.bincount(rows, minlength=n)[rows])
    vals[rng.random(len(vals)) < 0.05] = 0.0   # stored zeros
    return O.from_triplets(n, n, rows, cols, vals)


HUBS = [(1000, 100, 4000),      # warp (cap 128), bitmap
        (1500, 200, 5000),      # warp (cap 256, 8 x 32 entries per lane), bitmap
        (2500, 40, 3000),       # warp (cap 64), bitmap
        (2000, 300, 6000),      # CTA (cap 512), bitmap
        (3000, 700, 8000),      # CTA (cap 1024), bitmap
        (4000, 1500, 8100),     # CTA (cap 2048), bitmap
        (5000, 3000, 8150),     # CTA (cap 4096), bitmap
        (6000, 100, 20000),     # warp (cap 128), hash
        (7000, 400, 20000),     # CTA, hash
        (8000, 2500, 20000),    # CTA (cap 4096), hash
        (9000, 6000, 20000),    # cap 8192 hash: global-memory working set
        (10000, 7000, 8180)]    # cap 8192 bitmap: global-memory working set


@pytest.mark.parametrize('order', [2, 4, 6])
def test_poly_assembly_all_classes(order):
    import paper_2508_17517_b200 as G
    A = hub_matrix(3, 20000, HUBS)
    rng = np.random.default_rng(order)
    p = O.Poly('arnoldi_coeff', order, order, coeffs=rng.standard_normal(order + 1))
    same(G.assemble_fixed_sparsity(dev_poly(p), dev_csr(A)), O.assemble_poly(p, A))


def test_neumann_assembly_all_classes():
    import paper_2508_17517_b200 as G
    A = hub_matrix(4, 20000, HUBS)
    d = O.diag_of(A)
    d[d == 0] = 1.0
    A = O._mk(A.nrows, A.ncols, A.ptr, A.col, A.val)
    p = O.Poly('neumann', 3, 3, coeffs=np.ones(4), diag_scale=1.0 / (d + 2.0))
    same(G.assemble_fixed_sparsity(dev_poly(p), dev_csr(A)), O.assemble_poly(p, A))


def test_masked_product_all_classes():
    import paper_2508_17517_b200 as G
    A = hub_matrix(5, 20000, HUBS)
    B = hub_matrix(6, 20000, HUBS[::-1])
    P = hub_matrix(7, 20000, HUBS)
    same(G.spgemm_fixed_sparsity(dev_csr(A), dev_csr(B), dev_csr(P)), O.spgemm_masked(A, B, P))


# pattern rows beyond the largest pow2 cap class (32 << 10 = 32768 entries):
# they share the top class, whose cap is the longest row (global-memory
# working set), so any row length assembles as in the reference
LONG_HUBS = [(30000, 33000, 60000),   # top class, just above 32768
             (40000, 50000, 70000),   # top class, cap = this row's length
             (20000, 20000, 50000)]   # cap 32768 class below it


@pytest.mark.parametrize('order', [2, 5])
def test_poly_assembly_rows_beyond_caps(order):
    import paper_2508_17517_b200 as G
    A = hub_matrix(8, 80000, LONG_HUBS)
    rng = np.random.default_rng(10 + order)
    p = O.Poly('arnoldi_coeff', order, order, coeffs=rng.standard_normal(order + 1))
    same(G.assemble_fixed_sparsity(dev_poly(p), dev_csr(A)), O.assemble_poly(p, A))
