"""The distributed (GpuTeam) device path on ONE GPU: an NCCL communicator of
one rank drives the same schedule as N ranks -- local partial reductions ->
ncclAllReduce -> device epilogue, and (forced) agglomeration with an
ncclAllGather.  Halo exchanges are empty with one rank; their plans are
checked bitwise on a gloo world of 2 in tests/test_team.py."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2103_07329_b200 import BlockVector, gen_poisson3d  # noqa: E402
from paper_2103_07329_b200.params import tree  # noqa: E402
from paper_2103_07329_b200.solvers import prepare  # noqa: E402
from paper_2103_07329_b200.team import GpuTeam  # noqa: E402

JAC = {"method": "Jacobi", "weight": "0.8"}
CHEB = {"method": "Chebyshev", "polynomial_order": "2"}
CASES = {
    "amg_pcg": {"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"},
                "pre_smoother": JAC, "post_smoother": JAC},
    "amg_bicgstab_mixed": {"solver": {"method": "BiCGStab"},
                           "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": "1",
                                              "mg_coarse_matrix_size": "100"},
                           "pre_smoother": CHEB, "post_smoother": CHEB},
    "jacobi_pcg": {"solver": {"method": "CG", "max_iters": "500"},
                   "preconditioner": {"method": "Jacobi"}},
    "amg_rbicgstab": {"solver": {"method": "RBiCGStab"}, "preconditioner": {"method": "MultiGrid"},
                      "pre_smoother": JAC, "post_smoother": JAC},
    "amg_pbicgstab": {"solver": {"method": "PBiCGStab"},
                      "preconditioner": {"method": "MultiGrid", "mg_coarse_matrix_size": "100"},
                      "pre_smoother": CHEB, "post_smoother": CHEB},
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("force", [None, 1, 2])
def test_team_of_one_matches_single_gpu(name, force, monkeypatch):
    # distributed plans keep the per-level coarse kernels: compare like with like
    from paper_2103_07329_b200 import amg
    monkeypatch.setattr(amg, "DENSE_TAIL_ROWS", 0)
    A, _ = gen_poisson3d(14, 13, 12)
    B = np.random.default_rng(3).uniform(-1, 1, (A.nrows, 4))
    roles = CASES[name]
    Xs = BlockVector.zeros(A.nrows, 4)
    ss = prepare(tree(roles), A).run(BlockVector.from_array(B), Xs)
    team = GpuTeam(agg_rows_per_rank=1, force_replicate_from=force)
    cs = prepare(tree(roles), A, team=team)
    assert cs.row_range == (0, A.nrows)
    Xd = BlockVector.zeros(A.nrows, 4)
    sd = cs.run(BlockVector.from_array(B), Xd)
    assert sd.iterations == ss.iterations and sd.all_converged
    # one rank: identical arithmetic (NCCL sum of one partial is the partial)
    np.testing.assert_array_equal(Xd.data, Xs.data)
    np.testing.assert_array_equal(sd.final_rel_residual, ss.final_rel_residual)
    team.close()


@pytest.mark.parametrize("name", ["amg_pcg", "amg_pbicgstab", "amg_bicgstab_mixed"])
def test_team_of_one_dense_tail_on_replicated_levels(name):
    """The collapsed V-cycle tail also runs in distributed plans when its level
    is replicated (agglomerated): a 1-rank team replicating from level 1 gives
    the single-GPU bits."""
    A, _ = gen_poisson3d(14, 13, 12)
    B = np.random.default_rng(4).uniform(-1, 1, (A.nrows, 4))
    roles = CASES[name]
    Xs = BlockVector.zeros(A.nrows, 4)
    ss = prepare(tree(roles), A).run(BlockVector.from_array(B), Xs)
    team = GpuTeam(agg_rows_per_rank=1, force_replicate_from=1)
    cs = prepare(tree(roles), A, team=team)
    Xd = BlockVector.zeros(A.nrows, 4)
    sd = cs.run(BlockVector.from_array(B), Xd)
    assert sd.iterations == ss.iterations and sd.all_converged
    np.testing.assert_array_equal(Xd.data, Xs.data)
    team.close()


def test_team_single_gpu_only_configs_raise():
    from paper_2103_07329_b200.errors import ConfigurationError
    A, _ = gen_poisson3d(6, 6, 6)
    team = GpuTeam()
    for roles in ({"solver": {"method": "Direct"}},
                  {"solver": {"method": "Gauss-Seidel"}},
                  {"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"}}):
        with pytest.raises(ConfigurationError):
            prepare(tree(roles), A, team=team)
    team.close()


@pytest.mark.parametrize("roles", [
    {"solver": {"method": "MultiGrid", "rel_tolerance": "1e-8", "max_iters": "60"},
     "pre_smoother": JAC, "post_smoother": JAC},
    {"solver": {"method": "Jacobi", "rel_tolerance": "1e-3", "max_iters": "300", "weight": "0.9"}},
    {"solver": {"method": "CG", "rel_tolerance": "1e-9"},
     "preconditioner": {"method": "Chebyshev", "polynomial_order": "3"}},
])
def test_team_of_one_other_families(roles):
    """MultiGrid-as-solver, stationary Jacobi and the Chebyshev preconditioner
    through the distributed code path (1-rank NCCL team) equal the single-GPU
    bits."""
    A, _ = gen_poisson3d(10, 9, 8)
    B = np.random.default_rng(6).uniform(-1, 1, (A.nrows, 2))
    Xs = BlockVector.zeros(A.nrows, 2)
    ss = prepare(tree(roles), A).run(BlockVector.from_array(B), Xs)
    team = GpuTeam(agg_rows_per_rank=1, force_replicate_from=1)
    Xd = BlockVector.zeros(A.nrows, 2)
    sd = prepare(tree(roles), A, team=team).run(BlockVector.from_array(B), Xd)
    assert sd.iterations == ss.iterations
    np.testing.assert_array_equal(Xd.data, Xs.data)
    team.close()


@pytest.mark.parametrize("name", ["amg_pcg", "amg_bicgstab_mixed", "amg_pbicgstab"])
def test_team_of_one_split_products_in_captured_graphs(name, monkeypatch):
    """The halo/compute overlap as the product captures it (exec mode 2: the
    body graph holds 4 gated iterations, the exchange on the communication
    stream joined back by events): with one rank there is no halo, so the
    test mode of the knob forces the split on a shrunken interior range --
    interior rows, then boundary rows, two partial dot sets.  Same iterations,
    X to roundoff (the split dot sums two partial sets)."""
    from paper_2103_07329_b200 import _lib, amg, team as T
    monkeypatch.setattr(amg, "DENSE_TAIL_ROWS", 0)
    monkeypatch.setattr(T, "interior_range", lambda blk, nown: (blk.nrows // 4,
                                                                 3 * blk.nrows // 4))
    A, _ = gen_poisson3d(14, 13, 12)
    B = np.random.default_rng(5).uniform(-1, 1, (A.nrows, 4))
    roles = CASES[name]
    Xs = BlockVector.zeros(A.nrows, 4)
    ss = prepare(tree(roles), A).run(BlockVector.from_array(B), Xs)
    _lib.set_option("halo_overlap", 2)
    try:
        team = GpuTeam(agg_rows_per_rank=1)
        cs = prepare(tree(roles), A, team=team)
        assert cs.layouts[0].interior[0] == (A.nrows // 4, 3 * A.nrows // 4)
        Xd = BlockVector.zeros(A.nrows, 4)
        sd = cs.run(BlockVector.from_array(B), Xd)
        sd2 = cs.run(BlockVector.from_array(B), BlockVector.zeros(A.nrows, 4))   # graph replay
    finally:
        _lib.set_option("halo_overlap", 1)
    assert sd.iterations == ss.iterations == sd2.iterations and sd.all_converged
    err = np.abs(Xd.data - Xs.data).max() / np.abs(Xs.data).max()
    assert err <= 1e-11, err
    team.close()
