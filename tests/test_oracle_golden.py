"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (oracle/gen_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2103_07329_b200.io import gen_poisson3d


def test_spmv_kernels_bitwise(golden_kernels):
    g = golden_kernels
    for key in g["spmv_cases"]:
        case = key.split("_")[0]
        x, b, y0 = g[case + "_x"], g[case + "_b"], g[case + "_y0"]
        for mode in range(4):
            y = y0.copy()
            O.csr_spmv(g[key + "_rp"], g[key + "_ci"], g[key + "_v"], x, y, mode,
                       b if mode == 3 else None)
            np.testing.assert_array_equal(y, g[f"{key}_out{mode}"], err_msg=f"{key} mode {mode}")


def test_vector_kernels_bitwise(golden_kernels):
    g = golden_kernels
    for key in g["vec_cases"]:
        v = {n: g[f"{key}_{n}"] for n in ("x", "y", "u", "v", "w", "z", "s", "a", "bb", "c")}
        t = v["y"].copy(); O.axpby(v["a"], v["x"], v["bb"], t)
        np.testing.assert_array_equal(t, g[key + "_axpby"])
        t = v["y"].copy(); O.add2_scaled(t, v["a"], v["u"], v["bb"], v["v"])
        np.testing.assert_array_equal(t, g[key + "_add2"])
        np.testing.assert_array_equal(O.dot_partial(v["x"], v["y"]), g[key + "_dot"])
        t = v["y"].copy()
        np.testing.assert_array_equal(O.fused_update_dot(v["a"], v["x"], v["bb"], t), g[key + "_ud_dot"])
        np.testing.assert_array_equal(t, g[key + "_ud_y"])
        t1, t2 = v["y"].copy(), v["w"].copy()
        O.fused_paired_update(t1, v["a"], v["u"], v["bb"], v["s"], t2, v["c"], v["x"])
        np.testing.assert_array_equal(t1, g[key + "_pu_y1"])
        np.testing.assert_array_equal(t2, g[key + "_pu_y2"])
        t = v["y"].copy()
        d1, d2 = O.fused_update_dot2(t, v["u"], v["c"], v["w"], v["z"])
        np.testing.assert_array_equal(t, g[key + "_ud2_y"])
        np.testing.assert_array_equal(d1, g[key + "_ud2_d1"])
        np.testing.assert_array_equal(d2, g[key + "_ud2_d2"])


def _golden_csr(g, pre):
    from oracle.oracle import Csr
    nr, nc = g[pre + "_shape"]
    return Csr(int(nr), int(nc), g[pre + "_rp"], g[pre + "_ci"], g[pre + "_v"])


def test_oracle_setup_matches_reference(golden_hier):
    from oracle.amg_setup import setup
    g = golden_hier
    for name in g["hier_cases"]:
        A = _golden_csr(g, f"{name}_A")
        th, agg, npth, cs, ml, mixed = g[f"{name}_params"]
        h = setup(A, th, int(agg), int(npth), int(cs), int(ml), bool(mixed))
        assert len(h.levels) == int(g[f"{name}_nlevels"]), name
        for l, lv in enumerate(h.levels):
            for tag in ("A", "P", "R"):
                blk = getattr(lv, tag)
                key = f"{name}_L{l}_{tag}"
                if blk is None:
                    assert key + "_rp" not in g
                    continue
                np.testing.assert_array_equal(blk.row_ptr, g[key + "_rp"], err_msg=key)
                np.testing.assert_array_equal(blk.col_idx.astype(np.int64),
                                              g[key + "_ci"].astype(np.int64), err_msg=key)
                assert blk.values.dtype == g[key + "_v"].dtype, key
                np.testing.assert_array_equal(blk.values, g[key + "_v"], err_msg=key)


def _solve_case(name, g):
    """Re-run a golden solve case through the oracle drivers."""
    from oracle.amg_setup import setup
    from oracle.oracle import Csr
    import oracle.gen_golden as GG
    grid, m, seed, roles = GG.SOLVE_CASES[name]
    Ab, _ = gen_poisson3d(*grid)
    A = Csr.of(Ab)
    B = g[f"{name}_B"]
    X = np.zeros_like(B)
    sp_ = roles["solver"]
    tol = float(sp_.get("rel_tolerance", 1e-8))
    pre = roles.get("preconditioner")
    precond = None
    if pre and pre["method"] == "Jacobi":
        precond = O.JacobiPrecond(A, float(pre.get("weight", 1.0)), int(pre.get("max_iters", 1)))
    elif pre and pre["method"] == "Gauss-Seidel":
        precond = O.SgsPrecond(A, pre.get("direction", "symmetric"), int(pre.get("max_iters", 1)))
    elif pre and pre["method"] == "MultiGrid":
        h = setup(A, coarse_size=int(pre.get("mg_coarse_matrix_size", 500)),
                  agg_num_levels=int(pre.get("mg_agg_num_levels", 0)),
                  num_paths=int(pre.get("mg_num_paths", 1)),
                  mixed=bool(int(pre.get("mg_mixed_precision", 0))))
        def spec(r):
            d = roles.get(r)
            if d is None:                     # reference default: symmetric hybrid GS
                return ("sgs", "symmetric", 1)
            if d["method"] == "Gauss-Seidel":
                return ("sgs", d.get("direction", "symmetric"), int(d.get("max_iters", 1)))
            if d["method"] == "Jacobi":
                return ("jacobi", float(d.get("weight", 1.0)), int(d.get("max_iters", 1)))
            return ("chebyshev", int(d.get("polynomial_order", 2)))
        precond = O.MultiGrid(h, spec("pre_smoother"), spec("post_smoother"))
    elif pre and pre["method"] == "Chebyshev":
        precond = O.ChebPrecond(A, int(pre.get("polynomial_order", 2)))
    method = sp_["method"]
    iters = int(sp_.get("max_iters", 100))
    if method == "Direct":
        return O.direct_solve(A, B, X), X
    if method in ("MultiGrid", "Jacobi", "Gauss-Seidel"):
        if method == "MultiGrid":
            h = setup(A, coarse_size=int(sp_.get("mg_coarse_matrix_size", 500)))
            step = O.mg_step(O.MultiGrid(h, _spec(roles, "pre_smoother"),
                                         _spec(roles, "post_smoother")))
        elif method == "Jacobi":
            step = O.jacobi_step(A, float(sp_.get("weight", 1.0)))
        else:
            step = O.sgs_step(A, sp_.get("direction", "symmetric"))
        return O.stationary_solve(A, B, X, step, tol, iters), X
    drv = {"CG": O.cg_solve, "BiCGStab": O.bicgstab_solve, "RBiCGStab": O.rbicgstab_solve,
           "PBiCGStab": O.pbicgstab_solve}[method]
    st = drv(A, B, X, precond, tol, iters)
    return st, X


def _spec(roles, r):
    d = roles.get(r)
    if d is None:                     # reference default: symmetric hybrid GS
        return ("sgs", "symmetric", 1)
    if d["method"] == "Gauss-Seidel":
        return ("sgs", d.get("direction", "symmetric"), int(d.get("max_iters", 1)))
    if d["method"] == "Jacobi":
        return ("jacobi", float(d.get("weight", 1.0)), int(d.get("max_iters", 1)))
    return ("chebyshev", int(d.get("polynomial_order", 2)))


def _cases():
    import oracle.gen_golden as GG
    return list(GG.SOLVE_CASES)


@pytest.mark.parametrize("name", _cases())
def test_oracle_solves_match_reference(golden_solves, name):
    g = golden_solves
    st, X = _solve_case(name, g)
    assert st.iterations == int(g[f"{name}_iters"])
    # 1x1 topology: the oracle replays the reference arithmetic exactly
    np.testing.assert_array_equal(X, g[f"{name}_X"])
    np.testing.assert_array_equal(st.final_rel_residual, g[f"{name}_rel"])
    np.testing.assert_array_equal(np.array(st.residual_history), g[f"{name}_hist"])


def test_generator_matches_reference():
    from mrs_testutil import load_golden
    g = load_golden("generators.npz")
    for dims in ((2, 1, 1), (3, 4, 5), (8, 8, 8)):
        A, b = gen_poisson3d(*dims)
        key = "poisson_%dx%dx%d" % dims
        np.testing.assert_array_equal(A.row_ptr, g[key + "_rp"])
        np.testing.assert_array_equal(A.col_idx, g[key + "_ci"])
        assert A.col_idx.dtype == g[key + "_ci"].dtype
        np.testing.assert_array_equal(A.values, g[key + "_v"])
        np.testing.assert_array_equal(b.data, g[key + "_b"])


def test_oracle_eig_bounds_match_reference():
    from mrs_testutil import load_golden
    from oracle.oracle import Csr
    g = load_golden("eig.npz")
    A, _ = gen_poisson3d(9, 8, 7)
    Ao = Csr.of(A)
    assert tuple(O.estimate_eig_bounds(Ao, Ao.diagonal())) == tuple(g["p7_987"])
    A32 = Csr(Ao.nrows, Ao.ncols, Ao.row_ptr, Ao.col_idx, Ao.values.astype(np.float32))
    assert tuple(O.estimate_eig_bounds(A32, A32.diagonal())) == tuple(g["p7_987_f32"])
    I = Csr.from_scipy(np.eye(32))
    assert tuple(O.estimate_eig_bounds(I, I.diagonal())) == tuple(g["eye32"])
