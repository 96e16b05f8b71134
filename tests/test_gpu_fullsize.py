"""Parity at BASELINE.json's full sizes, against the reference's own outputs.

* C1 / C2 / C3 at full size and the C4 operator family (27-point anisotropic,
  24^3 .. 256^3, the last = BASELINE config 4): the device solve vs the reference run on the same seeded
  inputs (tests/golden/full_<case>.npz, written by oracle/gen_golden.py
  ``fullsize`` with the reference itself): iterations within +-1 (north
  star), every column's final relative residual <= tol, the strided X sample
  within 1e-6 of the reference's relative to the column's max, the residual
  history within 1e-5 relative over the common iterations; the hierarchy the
  device uploads hashes equal to the reference's, level by level (also on
  CPU: tests/test_fullsize_golden.py).
* C5 (n = 2^22, ~67 M entries): the device SpMM (slab-compressed 16-bit and
  32-bit columns, f64 and f32 values, m = 8) bitwise equals the oracle's C
  restatement of the reference kernel on the full matrix.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from mrs_testutil import GOLDEN, load_golden  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2103_07329_b200 import BlockVector, gen_poisson3d, kernels as K  # noqa: E402
from paper_2103_07329_b200.io import gen_random_sdd, gen_stencil27_aniso  # noqa: E402
from paper_2103_07329_b200.params import tree  # noqa: E402
from paper_2103_07329_b200.solvers import prepare  # noqa: E402

JAC = {"method": "Jacobi", "weight": "0.8"}
CHEB = {"method": "Chebyshev", "polynomial_order": "2"}
AMG_PCG = {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
           "preconditioner": {"method": "MultiGrid"},
           "pre_smoother": JAC, "post_smoother": JAC}
ROLES = {
    "c1": {"solver": {"method": "CG", "rel_tolerance": "1e-8", "max_iters": "1000"},
           "preconditioner": {"method": "Jacobi"}},
    "c2": AMG_PCG,
    "c3": {"solver": {"method": "BiCGStab", "rel_tolerance": "1e-8"},
           "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": "1"},
           "pre_smoother": CHEB, "post_smoother": CHEB},
    "c4_24": AMG_PCG, "c4_32": AMG_PCG, "c4_64": AMG_PCG, "c4_128": AMG_PCG,
    "c4_256": AMG_PCG,          # BASELINE config 4 at full size (449 M nnz, 17 levels)
}
CASES = [c for c in ROLES if os.path.exists(os.path.join(GOLDEN, f"full_{c}.npz"))]


def _sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def _matrix(g):
    grid = int(g["grid"])
    if str(g["kind"]) == "p7":
        return gen_poisson3d(grid, grid, grid)[0]
    return gen_stencil27_aniso(grid, seed=4)


@pytest.mark.parametrize("name", CASES)
def test_full_size_solve_vs_reference(name):
    g = load_golden(f"full_{name}.npz")
    A = _matrix(g)
    m = int(g["m"])
    B = np.random.default_rng(int(g["seed"])).uniform(-1.0, 1.0, (A.nrows, m))
    X = BlockVector.zeros(A.nrows, m)
    cs = prepare(tree(ROLES[name]), A)
    # the uploaded hierarchy is the reference's, level by level (SHA-256 of
    # row_ptr / col_idx / values of A, P, R)
    if "nlevels" in g.files:
        assert cs.hierarchy.nlevels == int(g["nlevels"])
        for l, lv in enumerate(cs.hierarchy.levels):
            for tag in ("A", "P", "R"):
                blk = getattr(lv, tag)
                if blk is not None:
                    got = [_sha(blk.row_ptr.astype(np.int64)),
                           _sha(blk.col_idx.astype(np.int64)), _sha(blk.values)]
                    assert got == list(g[f"L{l}_{tag}_sha"]), (name, l, tag)
    st = cs.run(BlockVector.from_array(B), X)
    it_ref = int(g["iters"])
    assert abs(st.iterations - it_ref) <= 1, (st.iterations, it_ref)
    assert st.all_converged and np.all(st.final_rel_residual <= 1e-8)
    rows = g["rows"]
    xr = g["X_rows"]
    err = np.abs(X.data[rows] - xr).max(axis=0) / np.abs(xr).max(axis=0)
    assert err.max() <= 1e-6, err
    hist_ref = g["hist"]
    k = min(len(st.residual_history), len(hist_ref))
    np.testing.assert_allclose(np.array(st.residual_history[:k]), hist_ref[:k], rtol=1e-5)
    # the final relative residuals are at the same level as the reference's
    np.testing.assert_allclose(st.final_rel_residual, g["rel"], rtol=0.5 if
                               st.iterations == it_ref else 10.0)


@pytest.fixture(scope="module")
def c5():
    return gen_random_sdd()


@pytest.mark.parametrize("slab", [True, False])
@pytest.mark.parametrize("vdt", [np.float64, np.float32])
def test_full_size_c5_spmm_bitwise(c5, slab, vdt):
    A = c5
    m = 8
    vals = A.values.astype(vdt)
    D = K.DeviceCsr(A.row_ptr, A.col_idx, vals, A.nrows, A.ncols, slab=slab)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (A.ncols, m))
    b = rng.uniform(-1, 1, (A.nrows, m))
    y = torch.empty(A.nrows, m, dtype=torch.float64, device="cuda")
    K.csr_spmv(D, None, None, torch.from_numpy(x).cuda(), y, K.MODE_RSUB, torch.from_numpy(b).cuda())
    ref = np.empty_like(b)
    O.csr_spmv(A.row_ptr, A.col_idx, vals, x, ref, O.MODE_RSUB, b)
    np.testing.assert_array_equal(y.cpu().numpy(), ref)
