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
