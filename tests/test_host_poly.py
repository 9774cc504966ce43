"""CPU tests of the host-side dense Krylov algebra of the GPU package (runs
on the device-built Hessenberg block): coefficients, harmonic Ritz roots,
Leja order and the residual history, against the oracle restatement."""

import numpy as np
import pytest

from oracle import airg_oracle as O
from paper_2508_17517_b200 import gmres_poly as GP


def _hess(seed, n=60, m=30, shift=2.0):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n)) * 0.3 + shift * np.eye(n)
    A = O.from_triplets(n, n, *np.nonzero(M), M[np.nonzero(M)])
    b = O.uniform_unit(n, seed)
    return O.arnoldi(A, b, m)


@pytest.mark.parametrize('seed', range(6))
def test_coefficients_identical_to_oracle(seed):
    H, k, beta = _hess(seed, m=5)
    mine = GP.coeffs_from_hessenberg(H, k, beta, 4)
    ref = O.arnoldi_coeffs_from_H(H, k, beta, 4)
    assert mine.coeffs.tobytes() == ref.coeffs.tobytes()
    assert mine.effective_order == ref.effective_order
    assert mine.residual_history == ref.history


@pytest.mark.parametrize('seed', range(6))
def test_newton_roots_and_leja_order_match_oracle(seed):
    H, k, beta = _hess(seed, m=30)
    mine = GP.roots_from_hessenberg(H, k, beta, 29)
    ref = O.newton_roots_from_H(H, k, beta, 29)
    assert mine.effective_order == ref.effective_order
    assert len(mine.roots) == len(ref.roots)
    assert np.allclose(mine.roots, ref.roots, rtol=1e-12, atol=0)
    # diagnostic history: Givens sweep vs per-step least squares
    assert np.allclose(mine.residual_history, ref.history, rtol=1e-8, atol=1e-14)


def test_newton_units_encoding():
    roots = np.array([3.0 + 0j, 1.0 + 2.0j, 1.0 - 2.0j, 0.5 + 0j])
    t, p1, p2 = GP.newton_units(roots)
    assert list(t) == [0, 1, 0]
    assert p1.tolist() == [3.0, 2.0, 0.5]
    assert p2[1] == 5.0
