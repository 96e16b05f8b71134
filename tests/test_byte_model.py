"""SURVEY.md 8(d) minimal byte model (byte_model.py) against hand counts."""

import numpy as np

from paper_2103_07329_b200 import _lib
from paper_2103_07329_b200.amg import setup
from paper_2103_07329_b200.byte_model import iteration_bytes_minimal, mat_bytes
from paper_2103_07329_b200.io import gen_poisson3d


def _desc(method, precond, pre=None, post=None, sweeps=1):
    d = _lib.mrs_plan_desc()
    d.method, d.precond, d.pc_sweeps, d.pc_weight, d.mg_cycles = method, precond, sweeps, 1.0, 1
    if pre is not None:
        d.pre, d.post = pre, post
    return d


def test_jacobi_pcg_and_mat_bytes():
    A = gen_poisson3d(10, 9, 8)[0]          # 720 rows: u16 columns
    n, m = A.nrows, 4
    assert mat_bytes(A) == A.nnz * (8 + 2) + (n + 1) * 4
    got = iteration_bytes_minimal(_desc(_lib.METHOD_CG, _lib.PC_JACOBI), [(A, None, None)], m)
    assert got == mat_bytes(A) + 11 * n * m * 8 + 16 * n


def test_amg_pcg_jacobi_vcycle_by_hand():
    A = gen_poisson3d(12, 12, 12)[0]
    h = setup(A)
    lv = [(l.A, l.P, l.R) for l in h.levels]
    m = 8
    jac = _lib.mrs_smoother(_lib.SMOOTH_JACOBI, 1, 0.8, 0, 0)
    got = iteration_bytes_minimal(_desc(_lib.METHOD_CG, _lib.PC_MG, jac, jac), lv, m)
    want = mat_bytes(lv[0][0]) + 13 * A.nrows * m * 8
    for l in range(len(lv) - 1):
        n, nc = lv[l][0].nrows, lv[l + 1][0].nrows
        V, Vc = n * m * 8, nc * m * 8
        want += (2 * V + 8 * n) + (mat_bytes(lv[l][0]) + 3 * V)          # pre, residual
        want += mat_bytes(lv[l][2]) + V + Vc + mat_bytes(lv[l][1]) + Vc + 2 * V
        want += mat_bytes(lv[l][0]) + 3 * V + 8 * n                      # post
    nL = lv[-1][0].nrows
    want += nL * nL * 8 + 2 * nL * m * 8
    assert got == want


def test_chebyshev2_matches_survey_counts():
    """Chebyshev order 2: pre mat + 5V + 16n, post 2 mat + 9V + 16n (8(d))."""
    from paper_2103_07329_b200.byte_model import _smoother_bytes
    A = gen_poisson3d(8, 8, 8)[0]
    n, V = A.nrows, A.nrows * 4 * 8
    ch = _lib.mrs_smoother(_lib.SMOOTH_CHEBYSHEV, 1, 0.0, 2, 0)
    assert _smoother_bytes(ch, A, n, V, pre=True) == mat_bytes(A) + 5 * V + 16 * n
    assert _smoother_bytes(ch, A, n, V, pre=False) == 2 * mat_bytes(A) + 9 * V + 16 * n
