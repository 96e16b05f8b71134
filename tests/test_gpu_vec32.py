"""fp32-vector V-cycle (``mg_vector_precision = fp32``; north star: "mixed
precision with an fp32 preconditioner").

An EXTENSION of the reference, whose vectors are always fp64 (its mixed mode
only stores level >= 1 matrix values in fp32, amg.py:291-307): the block
vectors of the V-cycle's levels 1 .. (collapsed tail or coarsest) - 1 are
float32 on the device -- loads widened, fp64 accumulation, stores rounded --
while the Krylov vectors and level 0 stay fp64.  Checked against
(a) the fp64 device solve of the same system: iterations within +-1, every
column converged, X within 1e-6; (b) the oracle's restatement of the same
rounding (oracle.MultiGridVec32): iterations within +-1, X within 1e-6;
(c) the plan's byte model, which must drop.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2103_07329_b200 import BlockVector, gen_poisson3d  # noqa: E402
from paper_2103_07329_b200.errors import ConfigurationError  # noqa: E402
from paper_2103_07329_b200.io import gen_stencil27_aniso  # noqa: E402
from paper_2103_07329_b200.params import tree  # noqa: E402
from paper_2103_07329_b200.solvers import prepare  # noqa: E402

JAC = {"method": "Jacobi", "weight": "0.8"}
CHEB = {"method": "Chebyshev", "polynomial_order": "2"}


def roles(solver, smoother, vprec, mixed="0"):
    return {"solver": {"method": solver, "rel_tolerance": "1e-8"},
            "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": mixed,
                               "mg_vector_precision": vprec},
            "pre_smoother": smoother, "post_smoother": smoother}


CASES = {
    "c3_shrunk": (lambda: gen_poisson3d(40, 40, 40)[0], 16, "BiCGStab", CHEB, "1"),
    "c2_shrunk": (lambda: gen_poisson3d(32, 32, 32)[0], 8, "CG", JAC, "0"),
    "s27": (lambda: gen_stencil27_aniso(24, seed=4), 8, "CG", JAC, "0"),
    "rbicgstab_m4": (lambda: gen_poisson3d(24, 24, 24)[0], 4, "RBiCGStab", CHEB, "0"),
    "cg_m1": (lambda: gen_poisson3d(24, 24, 24)[0], 1, "CG", JAC, "0"),
}


def solve(A, B, r):
    cs = prepare(tree(r), A)
    X = BlockVector.zeros(A.nrows, B.shape[1])
    st = cs.run(BlockVector.from_array(B), X)
    return cs, st, X.data


@pytest.mark.parametrize("case", list(CASES))
def test_vec32_matches_fp64_solve(case):
    mk, m, solver, sm, mixed = CASES[case]
    A = mk()
    B = np.random.default_rng(7).uniform(-1, 1, (A.nrows, m))
    cs64, st64, X64 = solve(A, B, roles(solver, sm, "fp64", mixed))
    cs32, st32, X32 = solve(A, B, roles(solver, sm, "fp32", mixed))
    assert abs(st32.iterations - st64.iterations) <= 1, (st32.iterations, st64.iterations)
    assert st32.all_converged and np.all(st32.final_rel_residual <= 1e-8)
    err = np.abs(X32 - X64).max(axis=0) / np.abs(X64).max(axis=0)
    assert err.max() <= 1e-6, err
    p32, p64 = cs32.plan_factory(m), cs64.plan_factory(m)
    assert p32.iteration_bytes < p64.iteration_bytes


@pytest.mark.parametrize("case", ["c2_shrunk", "c3_shrunk"])
def test_vec32_matches_rounding_oracle(case, monkeypatch):
    """The device's fp32 V-cycle vs its numpy restatement (per-level kernels:
    no collapsed tail, so the fp32 levels run down to the coarsest)."""
    from paper_2103_07329_b200 import amg
    from oracle.amg_setup import setup as osetup
    monkeypatch.setattr(amg, "DENSE_TAIL_ROWS", 0)
    mk, m, solver, sm, mixed = CASES[case]
    A = mk()
    B = np.random.default_rng(8).uniform(-1, 1, (A.nrows, m))
    cs, st, X = solve(A, B, roles(solver, sm, "fp32", mixed))
    Ao = O.Csr.of(A)
    h = osetup(Ao, mixed=bool(int(mixed)))
    spec = ("jacobi", 0.8, 1) if sm is JAC else ("chebyshev", 2)
    mg = O.MultiGridVec32(h, spec, spec)
    Xo = np.zeros_like(B)
    drv = O.cg_solve if solver == "CG" else O.bicgstab_solve
    so = drv(Ao, B, Xo, mg, 1e-8, 100)
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    err = np.abs(X - Xo).max(axis=0) / np.abs(Xo).max(axis=0)
    assert err.max() <= 1e-6, err


def test_vec32_unsupported_combinations_raise():
    A = gen_poisson3d(12, 12, 12)[0]
    B = np.random.default_rng(1).uniform(-1, 1, (A.nrows, 3))
    with pytest.raises(ConfigurationError):          # m not a power of two
        solve(A, B, roles("CG", JAC, "fp32"))
    with pytest.raises(ConfigurationError):          # pipelined: needs a linear M
        solve(A, B[:, :2].copy(), roles("PBiCGStab", JAC, "fp32"))
    r = roles("CG", JAC, "fp32")
    del r["pre_smoother"], r["post_smoother"]         # default Gauss-Seidel smoothing
    with pytest.raises(ConfigurationError):
        solve(A, B[:, :2].copy(), r)
    from paper_2103_07329_b200.team import GpuTeam
    team = GpuTeam()
    with pytest.raises(ConfigurationError):          # distributed plans stay fp64
        prepare(tree(roles("CG", JAC, "fp32")), A, team=team).run(
            BlockVector.from_array(B[:, :2].copy()), BlockVector.zeros(A.nrows, 2))
    team.close()


# ---- fp32_all: level 0 of the V-cycle on float vectors too (plan vec32 = 2) ----

@pytest.mark.parametrize("case", list(CASES))
def test_vec32_all_matches_fp64_solve(case):
    """The whole preconditioner on float vectors (the Krylov residual rounded on
    entry, the result widened on exit): iterations within +-1 of the fp64 solve,
    every column converged to 1e-8 (true fp64 residual), X within 1e-6.  (No byte
    claim: the two conversion passes and the separate (r, z) dot cost about what
    the float level-0 kernels save -- DESIGN.md section 5.)"""
    mk, m, solver, sm, mixed = CASES[case]
    A = mk()
    B = np.random.default_rng(7).uniform(-1, 1, (A.nrows, m))
    cs64, st64, X64 = solve(A, B, roles(solver, sm, "fp64", mixed))
    csa, sta, Xa = solve(A, B, roles(solver, sm, "fp32_all", mixed))
    assert abs(sta.iterations - st64.iterations) <= 1, (sta.iterations, st64.iterations)
    assert sta.all_converged and np.all(sta.final_rel_residual <= 1e-8)
    err = np.abs(Xa - X64).max(axis=0) / np.abs(X64).max(axis=0)
    assert err.max() <= 1e-6, err


@pytest.mark.parametrize("case", ["c2_shrunk", "c3_shrunk"])
def test_vec32_all_matches_rounding_oracle(case, monkeypatch):
    from paper_2103_07329_b200 import amg
    from oracle.amg_setup import setup as osetup
    monkeypatch.setattr(amg, "DENSE_TAIL_ROWS", 0)
    mk, m, solver, sm, mixed = CASES[case]
    A = mk()
    B = np.random.default_rng(8).uniform(-1, 1, (A.nrows, m))
    cs, st, X = solve(A, B, roles(solver, sm, "fp32_all", mixed))
    Ao = O.Csr.of(A)
    h = osetup(Ao, mixed=bool(int(mixed)))
    spec = ("jacobi", 0.8, 1) if sm is JAC else ("chebyshev", 2)
    mg = O.MultiGridVec32(h, spec, spec, level0=True)
    Xo = np.zeros_like(B)
    drv = O.cg_solve if solver == "CG" else O.bicgstab_solve
    so = drv(Ao, B, Xo, mg, 1e-8, 100)
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    err = np.abs(X - Xo).max(axis=0) / np.abs(Xo).max(axis=0)
    assert err.max() <= 1e-6, err


def test_vec32_all_multigrid_solver_is_rejected():
    """MultiGrid as the SOLVER iterates on the fp64 X itself: no float level 0."""
    A = gen_poisson3d(12, 12, 12)[0]
    B = np.random.default_rng(1).uniform(-1, 1, (A.nrows, 2))
    r = {"solver": {"method": "MultiGrid", "rel_tolerance": "1e-8", "mg_vector_precision": "fp32_all"},
         "pre_smoother": JAC, "post_smoother": JAC}
    with pytest.raises(ConfigurationError):
        solve(A, B, r)
