"""Collapsed V-cycle tail (amg.vcycle_tail_operator): the dense operator T_l
equals the sub-V-cycle from level l (zero guess) of the oracle restatement of
solvers.MultiGrid (solvers.py:651-664) on random right-hand sides.  CPU only:
T_l is setup-phase host code.  The device side (one dense launch instead of
the per-level kernels, same iterations as the reference) is covered in
tests/test_gpu_solvers.py."""

import numpy as np
import pytest

from oracle import oracle as O
from oracle.amg_setup import setup as osetup
from paper_2103_07329_b200 import _lib
from paper_2103_07329_b200.amg import (AmgParams, dense_tail_level, estimate_eig_bounds, setup,
                                       vcycle_tail_operator, coarse_inverse)
from paper_2103_07329_b200.io import gen_poisson3d


def _jac(w, s=1):
    return _lib.mrs_smoother(_lib.SMOOTH_JACOBI, s, w, 0, 0)


def _cheb(order):
    return _lib.mrs_smoother(_lib.SMOOTH_CHEBYSHEV, 1, 0.0, order, 0)


@pytest.mark.parametrize("mixed", [False, True])
@pytest.mark.parametrize("smoother", ["jacobi", "jacobi2", "cheb2", "cheb3", "sgs", "sgs_fwd2"])
def test_tail_operator_matches_oracle_vcycle(mixed, smoother):
    A, _ = gen_poisson3d(18, 17, 16)
    h = setup(A, AmgParams(coarse_matrix_size=40), mixed_precision=mixed)
    assert h.nlevels >= 4
    cheb = smoother.startswith("cheb")
    bounds = [estimate_eig_bounds(lv.A) if cheb and l < h.nlevels - 1 else None
              for l, lv in enumerate(h.levels)]
    levels = [(lv.A, lv.P, lv.R, bounds[l]) for l, lv in enumerate(h.levels)]
    inv = coarse_inverse(h.coarsest.A)
    spec = {"jacobi": (_jac(0.8), ("jacobi", 0.8, 1)), "jacobi2": (_jac(0.7, 2), ("jacobi", 0.7, 2)),
            "cheb2": (_cheb(2), ("chebyshev", 2)), "cheb3": (_cheb(3), ("chebyshev", 3)),
            "sgs": (_lib.mrs_smoother(_lib.SMOOTH_SGS, 1, 0.0, 0, 0), ("sgs", "symmetric", 1)),
            "sgs_fwd2": (_lib.mrs_smoother(_lib.SMOOTH_SGS, 2, 0.0, 0, 1), ("sgs", "forward", 2)),
            }[smoother]
    ho = osetup(O.Csr.of(A), coarse_size=40, mixed=mixed)
    for l, lv in enumerate(ho.levels):
        lv.eig_bounds = bounds[l]
    mg = O.MultiGrid(ho, spec[1], spec[1])
    rng = np.random.default_rng(3)
    for start in range(1, h.nlevels - 1):
        T = vcycle_tail_operator(levels, start, spec[0], spec[0], inv)
        n = h.levels[start].A.nrows
        assert T.shape == (n, n)
        b = rng.uniform(-1, 1, (n, 3))
        x = np.zeros_like(b)
        mg.vcycle(start, b, x, True)
        err = np.abs(T @ b - x).max() / np.abs(x).max()
        assert err < 1e-11, (start, err)


def test_tail_level_choice_and_sgs():
    A, _ = gen_poisson3d(16, 16, 16)
    h = setup(A, AmgParams(coarse_matrix_size=40))
    levels = [(lv.A, lv.P, lv.R, None) for lv in h.levels]
    sizes = [lv.A.nrows for lv in h.levels]
    l = dense_tail_level(levels, 1000)
    assert 1 <= l < h.nlevels - 1 and sizes[l] <= 1000
    # the cost model only collapses where the per-level kernels cost more
    # than streaming the dense operator: never the huge levels
    assert dense_tail_level(levels, 10 ** 9) >= 1
    assert sizes[dense_tail_level(levels, 10 ** 9)] < 5000
    assert dense_tail_level(levels, 0) == -1
    assert dense_tail_level(levels, sizes[-1]) == -1      # only the coarsest fits: nothing to collapse
    bad = _lib.mrs_smoother(99, 1, 0.0, 0, 0)                 # unknown smoother kind
    assert vcycle_tail_operator(levels, l, bad, bad, coarse_inverse(h.coarsest.A)) is None
