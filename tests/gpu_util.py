"""Helpers shared by the GPU parity tests: move oracle objects to the device
package and back (test infrastructure only)."""

import numpy as np

from oracle import airg_oracle as O


def dev_csr(M):
    import paper_2508_17517_b200 as G
    return G.SparseMatrix.csr(M.nrows, M.ncols, M.ptr, M.col, M.val, check=False)


def host_csr(M):
    p, c, v = M.to_host()
    return O._mk(M.nrows, M.ncols, p, c, v)


def dev_poly(p):
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200.csr import VAL, to_dev
    ds = to_dev(p.diag_scale, VAL) if p.diag_scale is not None else None
    return G.PolySolver(p.kind, p.order, p.effective_order, coeffs=p.coeffs, roots=p.roots,
                        diag_scale=ds, residual_history=p.history)


def oracle_poly(p):
    ds = p.diag_scale.cpu().numpy() if p.diag_scale is not None else None
    return O.Poly(p.kind, p.order, p.effective_order, coeffs=p.coeffs, roots=p.roots,
                  diag_scale=ds, history=p.residual_history)


def upload_hierarchy(Hh):
    """Oracle hierarchy -> device Hierarchy (solve-path parity on identical operators)."""
    import paper_2508_17517_b200 as G
    from paper_2508_17517_b200.amg_setup import finalize_complexities
    levels = []
    for L in Hh.levels:
        split = G.CFSplit.from_labels(L.labels)
        levels.append(G.Level(R=dev_csr(L.R), P=dev_csr(L.P), A_ff=dev_csr(L.A_ff),
                              A_fc=dev_csr(L.A_fc), f_smoother=dev_poly(L.smoother), split=split,
                              n=L.n, nnz_A=L.nnz_A,
                              f_smoother_assembled=None if L.assembled is None
                              else dev_csr(L.assembled)))
    H = G.Hierarchy(levels=levels, coarsest_A=dev_csr(Hh.coarsest_A),
                    coarse_solver=dev_poly(Hh.coarse_solver), top_A=dev_csr(Hh.top_A),
                    truncated_at=Hh.truncated_at)
    return finalize_complexities(H)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def tonp(x):
    """Host copy of a solve result (numpy in -> numpy out, device in -> device out)."""
    return x if isinstance(x, np.ndarray) else x.cpu().numpy()
