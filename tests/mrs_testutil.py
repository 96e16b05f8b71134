"""Helpers shared by the test modules (imported as a top-level module;
pytest puts tests/ on sys.path)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def have_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def random_csr(n, ncols, per_row, rng, diag=3.0):
    """Random CSR block (sorted unique columns, optional diagonal) built
    without scipy.sparse.random (which is very slow for large shapes)."""
    import scipy.sparse as sp
    from paper_2103_07329_b200.core import CsrBlock
    k = rng.poisson(per_row, n)
    rows = np.repeat(np.arange(n, dtype=np.int64), k)
    cols = rng.integers(0, ncols, rows.size)
    vals = rng.standard_normal(rows.size)
    A = sp.csr_matrix((vals, (rows, cols)), shape=(n, ncols))
    if diag and n == ncols:
        A = A + sp.eye(n) * diag
    A.sum_duplicates()
    return CsrBlock.from_scipy(A)
