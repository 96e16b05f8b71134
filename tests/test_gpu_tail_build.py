"""The collapsed V-cycle tail's dense operator built ON THE GPU
(solvers.tail_operator_device: the sub-hierarchy as a MultiGrid-as-solver
plan, one V-cycle applied to the unit vectors) against the host construction
(amg.vcycle_tail_operator, itself checked against the oracle's sub-V-cycle in
tests/test_dense_tail.py): same operator, only the dense coarse solve's
summation order differs."""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2103_07329_b200 import _lib, gen_poisson3d  # noqa: E402
from paper_2103_07329_b200 import solvers as S  # noqa: E402
from paper_2103_07329_b200.amg import (AmgParams, coarse_inverse, estimate_eig_bounds,  # noqa: E402
                                       setup, vcycle_tail_operator)
from paper_2103_07329_b200.io import gen_stencil27_aniso  # noqa: E402

JAC = _lib.mrs_smoother(_lib.SMOOTH_JACOBI, 1, 0.8, 0, 0)
JAC2 = _lib.mrs_smoother(_lib.SMOOTH_JACOBI, 2, 0.7, 0, 0)
CHEB = _lib.mrs_smoother(_lib.SMOOTH_CHEBYSHEV, 1, 0.0, 2, 0)
SGS = _lib.mrs_smoother(_lib.SMOOTH_SGS, 1, 0.0, 0, 0)


def hierarchy(A, mixed=False, cheb=False):
    h = setup(A, AmgParams(coarse_matrix_size=60), mixed_precision=mixed)
    levels = []
    for l, lv in enumerate(h.levels):
        b = estimate_eig_bounds(lv.A) if cheb and l < h.nlevels - 1 else None
        levels.append((lv.A, lv.P, lv.R, b))
    return h, levels, coarse_inverse(h.coarsest.A)


@pytest.mark.parametrize("case", ["poisson_jacobi", "poisson_jacobi2", "poisson_cheb_mixed",
                                  "s27_jacobi", "poisson_sgs"])
def test_device_tail_operator_matches_host(case):
    A = gen_stencil27_aniso(14, seed=4) if case.startswith("s27") else gen_poisson3d(18, 18, 18)[0]
    sm = {"poisson_jacobi": JAC, "poisson_jacobi2": JAC2, "poisson_cheb_mixed": CHEB,
          "s27_jacobi": JAC, "poisson_sgs": SGS}[case]
    h, levels, inv = hierarchy(A, mixed=case.endswith("mixed"), cheb=sm is CHEB)
    assert h.nlevels >= 3
    start = 1
    t0 = time.time()
    Th = vcycle_tail_operator(levels, start, sm, sm, inv)
    t1 = time.time()
    Td = S.tail_operator_device(levels, start, sm, sm, inv)
    t2 = time.time()
    assert Td.shape == Th.shape and Td.shape[0] == levels[start][0].nrows
    scale = np.abs(Th).max()
    assert np.abs(Td - Th).max() <= 1e-12 * scale, np.abs(Td - Th).max() / scale
    print(f"{case}: n_l {Th.shape[0]}  host {t1 - t0:.2f} s  device {t2 - t1:.2f} s")


def test_prepare_uses_the_device_builder_and_solves_agree(monkeypatch):
    """prepare() with the device-built tail and with the host-built tail: same
    iterations, solutions equal to rounding."""
    from paper_2103_07329_b200 import BlockVector
    from paper_2103_07329_b200.params import tree
    A = gen_poisson3d(32, 32, 32)[0]
    roles = {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
             "preconditioner": {"method": "MultiGrid"},
             "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
             "post_smoother": {"method": "Jacobi", "weight": "0.8"}}
    B = np.random.default_rng(3).uniform(-1, 1, (A.nrows, 8))
    res = {}
    for where in ("device", "host"):
        monkeypatch.setattr(S, "TAIL_BUILD", where)
        cs = S.prepare(tree(roles), A)
        X = BlockVector.zeros(A.nrows, 8)
        st = cs.run(BlockVector.from_array(B), X)
        res[where] = (st.iterations, X.data.copy())
    assert res["device"][0] == res["host"][0]
    err = np.abs(res["device"][1] - res["host"][1]).max() / np.abs(res["host"][1]).max()
    assert err <= 1e-10, err
