"""Device solves vs the reference (golden) and the oracle.

Parity contract (BASELINE.json north star): iteration counts within +-1 of
the reference on the same seeded inputs and hierarchy, every column's
recomputed final relative residual <= tol; here the arithmetic differs from
the reference only in the dot-reduction order, so solutions agree far
tighter (checked at 1e-6 relative to ||x||).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2103_07329_b200 import BlockVector, CsrBlock, gen_poisson3d  # noqa: E402
from paper_2103_07329_b200.errors import BreakdownError, ConfigurationError  # noqa: E402
from paper_2103_07329_b200.params import tree  # noqa: E402
from paper_2103_07329_b200.solvers import prepare, solve  # noqa: E402

import oracle.gen_golden as GG  # noqa: E402

CASES = list(GG.SOLVE_CASES)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["graph", "eager"])
def test_golden_solves(golden_solves, name, mode):
    g = golden_solves
    grid, m, seed, roles = GG.SOLVE_CASES[name]
    A, _ = gen_poisson3d(*grid)
    B = g[f"{name}_B"]
    cs = prepare(tree(roles), A, exec_mode=mode)
    X = BlockVector.zeros(A.nrows, m)
    st = cs.run(BlockVector.from_array(B), X)
    it_ref = int(g[f"{name}_iters"])
    tol = float(roles["solver"].get("rel_tolerance", 1e-8))
    assert abs(st.iterations - it_ref) <= 1, (st.iterations, it_ref)
    assert st.all_converged and np.all(st.final_rel_residual <= tol)
    Xr = g[f"{name}_X"]
    if st.iterations == it_ref:
        err = np.linalg.norm(X.data - Xr, axis=0) / np.linalg.norm(Xr, axis=0)
        assert err.max() < 1e-6, err
        h = np.array(st.residual_history)
        np.testing.assert_allclose(h, g[f"{name}_hist"], rtol=1e-5, atol=0.1 * tol)


def test_graph_and_eager_agree_bitwise():
    A, _ = gen_poisson3d(12, 12, 12)
    B = np.random.default_rng(3).uniform(-1, 1, (A.nrows, 4))
    roles = GG.SOLVE_CASES["c2_amg_pcg"][3]
    out = []
    for mode in ("graph", "eager", "graph"):
        X = BlockVector.zeros(A.nrows, 4)
        st = prepare(tree(roles), A, exec_mode=mode).run(BlockVector.from_array(B), X)
        out.append((st.iterations, X.data.copy()))
    assert out[0][0] == out[1][0] == out[2][0]
    np.testing.assert_array_equal(out[0][1], out[1][1])
    np.testing.assert_array_equal(out[0][1], out[2][1])


def test_rerun_same_prepared_solver_is_reproducible():
    A, b = gen_poisson3d(8, 8, 8)
    cs = prepare(tree({"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"},
                       "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
                       "post_smoother": {"method": "Jacobi", "weight": "0.8"}}), A)
    x1 = BlockVector.zeros(512, 1)
    s1 = cs.run(b, x1)
    x2 = BlockVector.zeros(512, 1)
    s2 = cs.run(b, x2)
    np.testing.assert_array_equal(x1.data, x2.data)
    assert s1.iterations == s2.iterations and s1.all_converged


def test_cg_two_by_two_exact():
    a = np.array([[4.0, 1.0], [1.0, 3.0]])
    x = BlockVector.zeros(2, 1)
    st = solve(tree({"solver": {"method": "CG", "rel_tolerance": "1e-14"}}),
               CsrBlock.from_dense(a), BlockVector.from_array([1.0, 2.0]), x)
    np.testing.assert_allclose(x.data[:, 0], [1 / 11, 7 / 11], rtol=1e-12)
    assert st.iterations <= 2 and st.all_converged


def test_bicgstab_identity_one_iteration():
    x = BlockVector.zeros(5, 2)
    b = np.arange(10.0).reshape(5, 2) + 1
    st = solve(tree({"solver": {"method": "BiCGStab"}}), CsrBlock.from_dense(np.eye(5)),
               BlockVector.from_array(b), x)
    assert st.iterations == 1
    np.testing.assert_allclose(x.data, b, rtol=1e-14)


def test_zero_rhs_zero_iterations():
    A, _ = gen_poisson3d(4, 4, 4)
    x = BlockVector.zeros(64, 2)
    st = solve(tree({"solver": {"method": "CG"}}), A, BlockVector.zeros(64, 2), x)
    assert st.iterations == 0 and st.all_converged
    np.testing.assert_array_equal(x.data, 0.0)


def test_zero_rhs_column_stays_zero():
    A, _ = gen_poisson3d(5, 5, 5)
    b = np.zeros((125, 2))
    b[:, 1] = np.random.default_rng(0).standard_normal(125)
    x = BlockVector.zeros(125, 2)
    st = solve(tree({"solver": {"method": "CG", "rel_tolerance": "1e-10"}}), A,
               BlockVector.from_array(b), x)
    assert st.all_converged
    np.testing.assert_array_equal(x.data[:, 0], 0.0)


def test_breakdown_raises_with_column():
    a = np.array([[1.0, 0.0], [0.0, -1.0]])
    with pytest.raises(BreakdownError) as ei:
        solve(tree({"solver": {"method": "CG"}}), CsrBlock.from_dense(a),
              BlockVector.from_array([1.0, 1.0]), BlockVector.zeros(2, 1))
    assert ei.value.column == 0


def test_nonzero_initial_guess_at_solution():
    A, b = gen_poisson3d(6, 6, 6)
    x = BlockVector.from_array(np.ones(216))
    st = solve(tree({"solver": {"method": "CG", "rel_tolerance": "1e-10"}}), A, b, x)
    assert st.iterations == 0


def test_max_iters_respected():
    A, _ = gen_poisson3d(10, 10, 10)
    B = np.random.default_rng(1).uniform(-1, 1, (1000, 2))
    x = BlockVector.zeros(1000, 2)
    st = solve(tree({"solver": {"method": "CG", "max_iters": "5"}}), A, BlockVector.from_array(B), x)
    assert st.iterations == 5 and not st.all_converged
    assert len(st.residual_history) == 6


def test_joint_equals_single_rhs():
    """Joint m-RHS solve equals m single-RHS solves (tests/test_acceptance.py:97-136)."""
    A, _ = gen_poisson3d(10, 10, 10)
    B = np.random.default_rng(5).uniform(-1, 1, (1000, 4))
    roles = {"solver": {"method": "BiCGStab", "rel_tolerance": "1e-10"},
             "preconditioner": {"method": "MultiGrid", "mg_coarse_matrix_size": "60"},
             "pre_smoother": {"method": "Chebyshev"}, "post_smoother": {"method": "Chebyshev"}}
    cs = prepare(tree(roles), A)
    X = BlockVector.zeros(1000, 4)
    cs.run(BlockVector.from_array(B), X)
    for j in range(4):
        xj = BlockVector.zeros(1000, 1)
        cs.run(BlockVector.from_array(B[:, j:j + 1]), xj)
        np.testing.assert_allclose(X.data[:, j], xj.data[:, 0], rtol=1e-10, atol=1e-12)


def test_device_tensor_run_matches_host_run():
    A, _ = gen_poisson3d(12, 12, 12)
    B = np.random.default_rng(2).uniform(-1, 1, (A.nrows, 8))
    cs = prepare(tree(GG.SOLVE_CASES["c2_amg_pcg"][3]), A)
    Xh = BlockVector.zeros(A.nrows, 8)
    s1 = cs.run(BlockVector.from_array(B), Xh)
    Bd = torch.from_numpy(B).cuda()
    Xd = torch.zeros_like(Bd)
    s2 = cs.run(Bd, Xd)
    assert s1.iterations == s2.iterations
    np.testing.assert_array_equal(Xd.cpu().numpy(), Xh.data)


def test_unsupported_configs_raise():
    A, _ = gen_poisson3d(4, 4, 4)
    # a Krylov solver as preconditioner / smoother is not on the device path
    with pytest.raises(ConfigurationError):
        prepare(tree({"solver": {"method": "CG"}, "preconditioner": {"method": "BiCGStab"}}), A)
    with pytest.raises(ConfigurationError):
        prepare(tree({"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"},
                      "pre_smoother": {"method": "BiCGStab"}}), A)
    # as in the reference (solvers.py:904-905, :953)
    with pytest.raises(ConfigurationError):
        prepare(tree({"solver": {"method": "MultiGrid"}, "preconditioner": {"method": "Jacobi"}}), A)
    with pytest.raises(ConfigurationError):
        prepare(tree({"solver": {"method": "Chebyshev"}}), A)


@pytest.mark.parametrize("mode", ["graph", "eager"])
def test_default_gauss_seidel_multigrid_matches_oracle(mode):
    """MultiGrid without explicit smoothers uses the reference default (one
    symmetric hybrid Gauss-Seidel sweep, solvers.py:609-612): iterations and
    history against the oracle restatement on a 24^3 problem."""
    from oracle import oracle as O
    from oracle.amg_setup import setup as osetup
    A, _ = gen_poisson3d(24, 24, 24)
    B = np.random.default_rng(21).uniform(-1, 1, (A.nrows, 4))
    roles = {"solver": {"method": "CG", "rel_tolerance": "1e-9"},
             "preconditioner": {"method": "MultiGrid"}}
    X = BlockVector.zeros(A.nrows, 4)
    st = prepare(tree(roles), A, exec_mode=mode).run(BlockVector.from_array(B), X)
    Ao = O.Csr.of(A)
    mg = O.MultiGrid(osetup(Ao), ("sgs", "symmetric", 1), ("sgs", "symmetric", 1))
    Xo = np.zeros_like(B)
    so = O.cg_solve(Ao, B, Xo, mg, 1e-9, 100)
    assert st.iterations == so.iterations and st.all_converged
    np.testing.assert_allclose(np.array(st.residual_history), np.array(so.residual_history),
                               rtol=1e-6, atol=1e-12)
    assert np.max(np.abs(X.data - Xo)) <= 1e-8 * np.max(np.abs(Xo))


VARIANTS = ("BiCGStab", "RBiCGStab", "PBiCGStab")


@pytest.mark.parametrize("method", VARIANTS)
def test_bicgstab_variant_names_and_merged(method):
    """SolveStats.method as the reference names it; merged=1 is bitwise the
    same iterate sequence for the reordered and pipelined forms
    (tests/test_solvers.py:461-471)."""
    A, b = gen_poisson3d(8, 8, 8)
    out = []
    for merged in ("0", "1"):
        x = BlockVector.zeros(512, 1)
        st = solve(tree({"solver": {"method": method, "merged": merged,
                                    "rel_tolerance": "1e-10"}}), A, b, x)
        assert st.method == method + ("/merged" if merged == "1" else "")
        assert st.all_converged
        out.append(x.data.copy())
    if method != "BiCGStab":
        np.testing.assert_array_equal(out[0], out[1])


@pytest.mark.parametrize("system", ["poisson16", "sdd150"])
def test_bicgstab_variant_equivalence(system):
    """tests/test_acceptance.py:139-171: the first 10 residual-history entries
    of the variants agree with the classical one within 1e-6 relative and the
    solutions within 1e-8."""
    rng = np.random.default_rng(11)
    if system == "poisson16":
        A, b = gen_poisson3d(16, 16, 16)
        B = b.data
    else:
        n = 150
        a = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.1)
        a += np.diag(np.abs(a).sum(axis=1) + 1.0)
        A, B = CsrBlock.from_dense(a), rng.standard_normal((n, 1))
    hist, sols = [], []
    for method, merged in (("BiCGStab", "0"), ("RBiCGStab", "0"), ("PBiCGStab", "0"),
                           ("BiCGStab", "1")):
        x = BlockVector.zeros(A.nrows, 1)
        st = solve(tree({"solver": {"method": method, "merged": merged, "rel_tolerance": "1e-10",
                                    "max_iters": "200"}}), A, BlockVector.from_array(B), x)
        assert st.all_converged
        hist.append(np.array([h[0] for h in st.residual_history[:11]]))
        sols.append(x.data.copy())
    for h, xv in zip(hist[1:], sols[1:]):
        k = min(len(h), len(hist[0]))
        assert np.max(np.abs(h[:k] - hist[0][:k]) / np.abs(hist[0][:k])) <= 1e-6
        assert np.max(np.abs(xv - sols[0])) <= 1e-8


@pytest.mark.parametrize("method", VARIANTS)
def test_bicgstab_variants_breakdown_column(method):
    """r0 orthogonal to A r0 in column 0 (tests/test_solvers.py:158-165)."""
    a = np.array([[0.0, 1.0], [1.0, 0.0]])
    b = np.array([[1.0, 3.0], [0.0, 4.0]])
    with pytest.raises(BreakdownError) as ei:
        solve(tree({"solver": {"method": method}}), CsrBlock.from_dense(a),
              BlockVector.from_array(b), BlockVector.zeros(2, 2))
    assert ei.value.column == 0


def test_pipelined_drift_check_raises(monkeypatch):
    """tests/test_solvers.py:176-185: with DRIFT_LIMIT below the rounding
    noise the device cross-check fires (InstabilityError), and the default
    limit is the reference's 1e3."""
    from paper_2103_07329_b200 import solvers as S
    from paper_2103_07329_b200.errors import InstabilityError
    assert S.DRIFT_LIMIT == 1e3
    A, b = gen_poisson3d(8, 8, 8)
    monkeypatch.setattr(S, "DRIFT_LIMIT", 1e-12)
    for mode in ("graph", "eager"):
        with pytest.raises(InstabilityError):
            prepare(tree({"solver": {"method": "PBiCGStab", "rel_tolerance": "1e-10"}}), A,
                    exec_mode=mode).run(b, BlockVector.zeros(512, 1))


@pytest.mark.parametrize("method", ["RBiCGStab", "PBiCGStab"])
def test_variants_multi_rhs_column_independence(method):
    """tests/test_acceptance.py:95-136 (criterion 2) for the reordered and
    pipelined forms: joint solves equal per-column solves within 1e-10."""
    A, _ = gen_poisson3d(16, 16, 16)
    B = np.random.default_rng(913).standard_normal((A.nrows, 4))
    cs = prepare(tree({"solver": {"method": method, "rel_tolerance": "0", "max_iters": "10"}}), A)
    X = BlockVector.zeros(A.nrows, 4)
    cs.run(BlockVector.from_array(B), X)
    for j in range(4):
        xj = BlockVector.zeros(A.nrows, 1)
        cs.run(BlockVector.from_array(B[:, j:j + 1].copy()), xj)
        assert np.max(np.abs(X.data[:, j] - xj.data[:, 0])) <= 1e-10


def test_amg_pbicgstab_iteration_budget():
    """tests/test_solvers.py:384-398: AMG (Chebyshev-2) PBiCGStab on 16^3
    converges within 20 iterations."""
    A, b = gen_poisson3d(16, 16, 16)
    x = BlockVector.zeros(16 ** 3, 1)
    st = solve(tree({"solver": {"method": "PBiCGStab", "rel_tolerance": "1e-8"},
                     "preconditioner": {"method": "MultiGrid", "mg_coarse_matrix_size": "500"},
                     "pre_smoother": {"method": "Chebyshev", "polynomial_order": "2"},
                     "post_smoother": {"method": "Chebyshev", "polynomial_order": "2"}}), A, b, x)
    assert st.all_converged and st.iterations <= 20


@pytest.mark.parametrize("m", [1, 2, 3, 16, 32, 64])
def test_rhs_counts_vs_oracle_iterations(m):
    from oracle import oracle as O
    from oracle.amg_setup import setup as osetup
    A, _ = gen_poisson3d(14, 13, 12)
    B = np.random.default_rng(m).uniform(-1, 1, (A.nrows, m))
    roles = {"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"},
             "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
             "post_smoother": {"method": "Jacobi", "weight": "0.8"}}
    X = BlockVector.zeros(A.nrows, m)
    st = prepare(tree(roles), A).run(BlockVector.from_array(B), X)
    Ao = O.Csr.of(A)
    mg = O.MultiGrid(osetup(Ao), ("jacobi", 0.8, 1), ("jacobi", 0.8, 1))
    Xo = np.zeros_like(B)
    so = O.cg_solve(Ao, B, Xo, mg, 1e-8, 100)
    assert abs(st.iterations - so.iterations) <= 1
    assert st.all_converged
    np.testing.assert_allclose(X.data, Xo, rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("roles", [GG.SOLVE_CASES["c2_amg_pcg_20"][3],
                                   GG.SOLVE_CASES["c3_amg_bicgstab_full_cheb3"][3],
                                   GG.SOLVE_CASES["c3_amg_bicgstab_mixed"][3],
                                   GG.SOLVE_CASES["amg_pcg_default_sgs"][3],
                                   {"solver": {"method": "CG", "rel_tolerance": "1e-9"},
                                    "preconditioner": {"method": "MultiGrid", "max_iters": "2"},
                                    "pre_smoother": {"method": "Jacobi", "weight": "0.7"},
                                    "post_smoother": {"method": "Chebyshev",
                                                      "polynomial_order": "2"}}])
@pytest.mark.parametrize("m", [1, 8, 16])
def test_dense_tail_matches_per_level_kernels(roles, m, monkeypatch):
    """The collapsed V-cycle tail (one dense launch for the levels <=
    DENSE_TAIL_ROWS rows) is the same operator as the per-level kernels:
    same iteration count, solutions equal to rounding, fewer launches."""
    from paper_2103_07329_b200 import amg
    A, _ = gen_poisson3d(24, 22, 20)
    B = np.random.default_rng(m).uniform(-1, 1, (A.nrows, m))
    out = {}
    for rows in (0, 2500):
        monkeypatch.setattr(amg, "DENSE_TAIL_ROWS", rows)
        cs = prepare(tree(roles), A)
        X = BlockVector.zeros(A.nrows, m)
        st = cs.run(BlockVector.from_array(B), X)
        assert st.all_converged
        out[rows] = (st.iterations, X.data.copy(), cs.plan_factory(m).kernels_per_iteration)
    assert out[0][0] == out[2500][0]
    np.testing.assert_allclose(out[2500][1], out[0][1], rtol=0, atol=1e-9 * np.abs(out[0][1]).max())
    assert out[2500][2] < out[0][2]


def _arrowhead_system(g=16, nlong=12, width=400, seed=5):
    """SPD Poisson-plus-arrowhead matrix: `nlong` rows coupled to `width`
    random columns each (symmetrised, diagonally dominant), so level 0 (and
    the coarse operators built from it) carry rows far longer than the mean."""
    import scipy.sparse as sp
    A, _ = gen_poisson3d(g, g, g)
    n = A.nrows
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in rng.choice(n, nlong, replace=False):
        js = rng.choice(n, width, replace=False)
        js = js[js != i]
        rows += [i] * len(js)
        cols += list(js)
    E = sp.csr_matrix((rng.uniform(-0.5, 0.5, len(rows)), (rows, cols)), shape=(n, n))
    E = E + E.T
    M = A.to_scipy() + E
    M = M + sp.diags(np.abs(E).sum(axis=1).A1)
    return CsrBlock.from_scipy(sp.csr_matrix(M))


@pytest.mark.parametrize("roles", [GG.SOLVE_CASES["c2_amg_pcg_20"][3],
                                   GG.SOLVE_CASES["c3_amg_bicgstab_full_cheb3"][3],
                                   GG.SOLVE_CASES["c3_amg_bicgstab_mixed"][3]])
@pytest.mark.parametrize("m", [1, 4, 8, 16, 3])
def test_long_row_ctas_bitwise(roles, m):
    """Rows far longer than their operator's mean are accumulated by whole
    CTAs (products in parallel, in-order fold; the SpMM itself is bitwise the
    lane path, test_gpu_kernels.py::test_spmv_long_rows_bitwise).  In a solve
    only the fused dots' CTA partition changes: same iterations, solutions
    equal to the last bits."""
    from paper_2103_07329_b200 import _lib
    A = _arrowhead_system()
    lens = np.diff(A.row_ptr)
    assert lens.max() > max(64, 4 * lens.mean())
    B = np.random.default_rng(m).uniform(-1, 1, (A.nrows, m))
    out = {}
    try:
        for split in (0, 1):
            _lib.set_option("spmm_long_split", split)
            cs = prepare(tree(roles), A)
            X = BlockVector.zeros(A.nrows, m)
            st = cs.run(BlockVector.from_array(B), X)
            out[split] = (st.iterations, X.data.copy(), np.array(st.residual_history))
    finally:
        _lib.set_option("spmm_long_split", 1)
    assert out[0][0] == out[1][0]
    np.testing.assert_allclose(out[1][1], out[0][1], rtol=0, atol=1e-12 * np.abs(out[0][1]).max())


@pytest.mark.parametrize("m", [8, 16, 3])
@pytest.mark.parametrize("mma", [0, 1])
def test_direct_solver_dense_kernels(m, mma):
    """Direct (dense inverse) solves through the dense-apply kernels: the FP64
    tensor-core kernel (n > 1024, m = 8 / 16) and the CUDA-core ones."""
    from paper_2103_07329_b200 import _lib
    A, _ = gen_poisson3d(12, 12, 12)
    B = np.random.default_rng(m).uniform(-1, 1, (A.nrows, m))
    try:
        _lib.set_option("dense_mma", mma)
        X = BlockVector.zeros(A.nrows, m)
        st = prepare(tree({"solver": {"method": "Direct"}}), A).run(BlockVector.from_array(B), X)
    finally:
        _lib.set_option("dense_mma", 1)
    ref = np.linalg.solve(A.to_dense(), B)
    np.testing.assert_allclose(X.data, ref, rtol=0, atol=1e-11 * np.abs(ref).max())
    assert st.iterations == 1 and np.all(st.converged)


@pytest.mark.parametrize("pc", [None, {"method": "Jacobi"}])
@pytest.mark.parametrize("max_iters", ["7", "500"])
def test_cg_loop_unroll_bitwise(pc, max_iters):
    """Short CG bodies are captured U times per trip of the WHILE node, the
    extra copies guarded by `stop`: iterations (also when max_iters cuts a
    trip short), history and X bitwise those of one copy per trip."""
    from paper_2103_07329_b200 import _lib
    A, _ = gen_poisson3d(16, 15, 14)
    B = np.random.default_rng(11).uniform(-1, 1, (A.nrows, 4))
    roles = {"solver": {"method": "CG", "rel_tolerance": "1e-9", "max_iters": max_iters}}
    if pc is not None:
        roles["preconditioner"] = pc
    out = {}
    try:
        for u in (1, 4, 3):
            _lib.set_option("loop_unroll", u)
            cs = prepare(tree(roles), A)
            X = BlockVector.zeros(A.nrows, 4)
            st = cs.run(BlockVector.from_array(B), X)
            out[u] = (st.iterations, X.data.copy(), np.array(st.residual_history))
    finally:
        _lib.set_option("loop_unroll", 4)
    for u in (4, 3):
        assert out[u][0] == out[1][0]
        np.testing.assert_array_equal(out[u][1], out[1][1])
        np.testing.assert_array_equal(out[u][2], out[1][2])
    if max_iters == "7":
        assert out[1][0] == 7


def test_coop_auto_on_27_point_operator():
    """The 27-point fine level (long uniform rows) takes the cooperative
    entry-load SpMM by default (spmm_coop = 2); same iterations and solution
    as the lane path."""
    from paper_2103_07329_b200 import _lib
    from paper_2103_07329_b200.io import gen_stencil27_aniso
    A = gen_stencil27_aniso(24, seed=4)
    B = np.random.default_rng(2).uniform(-1, 1, (A.nrows, 8))
    roles = {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
             "preconditioner": {"method": "MultiGrid"},
             "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
             "post_smoother": {"method": "Jacobi", "weight": "0.8"}}
    out = {}
    try:
        for mode in (0, 2):
            _lib.set_option("spmm_coop", mode)
            X = BlockVector.zeros(A.nrows, 8)
            st = prepare(tree(roles), A).run(BlockVector.from_array(B), X)
            assert st.all_converged
            out[mode] = (st.iterations, X.data.copy())
    finally:
        _lib.set_option("spmm_coop", 2)
    assert out[0][0] == out[2][0]
    np.testing.assert_allclose(out[2][1], out[0][1], rtol=0, atol=1e-9 * np.abs(out[0][1]).max())
