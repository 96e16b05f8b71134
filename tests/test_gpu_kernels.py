"""Device kernel plugin vs the reference's golden outputs and the C oracle.

SpMM and the element-wise vector kernels are bitwise equal to the reference
(same per-(row, column) operation order, no FMA).  Dots are reduced in a
different (blocked tree) order: compared at 1e-13 relative.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2103_07329_b200 import kernels as K  # noqa: E402
from paper_2103_07329_b200.core import CsrBlock  # noqa: E402

DEV = torch.device("cuda")

_TDT = {np.dtype(np.uint8): torch.uint8, np.dtype(np.uint16): torch.uint16,
        np.dtype(np.uint32): torch.uint32}


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def spmv_dev(rp, ci, v, x, y0, mode, b=None):
    y = T(y0)
    K.csr_spmv(T(rp.astype(np.int32)), T(ci), T(v), T(x), y, mode, T(b) if b is not None else None)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def test_spmv_golden_bitwise(golden_kernels):
    g = golden_kernels
    n = 0
    for key in g["spmv_cases"]:
        case = key.split("_")[0]
        x, b, y0 = g[case + "_x"], g[case + "_b"], g[case + "_y0"]
        for mode in range(4):
            y = spmv_dev(g[key + "_rp"], g[key + "_ci"], g[key + "_v"], x, y0, mode,
                         b if mode == 3 else None)
            np.testing.assert_array_equal(y, g[f"{key}_out{mode}"], err_msg=f"{key} mode {mode}")
            n += 1
    assert n >= 100


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8, 16, 32, 64])
@pytest.mark.parametrize("vdt", [np.float64, np.float32])
@pytest.mark.parametrize("width", [np.uint16, np.uint32])
def test_spmv_random_vs_oracle_bitwise(m, vdt, width, rng):
    from mrs_testutil import random_csr
    n = 3000 if width == np.uint16 else 70001
    blk = random_csr(n, n, 12.0, rng)
    ci = blk.col_idx.astype(width)
    v = blk.values.astype(vdt)
    x = rng.standard_normal((n, m))
    y0 = rng.standard_normal((n, m))
    b = rng.standard_normal((n, m))
    for mode in range(4):
        ref = y0.copy()
        O.csr_spmv(blk.row_ptr, ci, v, x, ref, mode, b)
        got = spmv_dev(blk.row_ptr, ci, v, x, y0, mode, b)
        np.testing.assert_array_equal(got, ref, err_msg=f"m={m} mode={mode}")


def test_spmv_unaligned_view_uses_generic_path(rng):
    n, m = 500, 4
    blk = CsrBlock.from_dense(rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.02))
    big = torch.zeros(n * m + 1, dtype=torch.float64, device=DEV)
    x = big[1:].view(n, m)                    # 8-byte aligned, not 16
    xh = rng.standard_normal((n, m))
    x.copy_(T(xh))
    y = torch.empty(n, m, dtype=torch.float64, device=DEV)
    K.csr_spmv(T(blk.row_ptr.astype(np.int32)), T(blk.col_idx), T(blk.values), x, y, 0)
    ref = np.empty((n, m))
    O.csr_spmv(blk.row_ptr, blk.col_idx, blk.values, xh, ref, 0)
    np.testing.assert_array_equal(y.cpu().numpy(), ref)


def test_spmv_rejects_alias_and_host(rng):
    from paper_2103_07329_b200.errors import InvalidArgumentError
    blk = CsrBlock.from_dense(np.eye(4))
    x = torch.ones(4, 1, dtype=torch.float64, device=DEV)
    with pytest.raises(InvalidArgumentError):
        K.csr_spmv(T(blk.row_ptr.astype(np.int32)), T(blk.col_idx), T(blk.values), x, x, 0)
    with pytest.raises(InvalidArgumentError):
        K.csr_spmv(T(blk.row_ptr.astype(np.int32)), T(blk.col_idx), T(blk.values),
                   x.cpu(), torch.empty(4, 1, dtype=torch.float64), 0)


def test_vector_kernels_golden(golden_kernels):
    g = golden_kernels
    for key in g["vec_cases"]:
        v = {nm: g[f"{key}_{nm}"] for nm in ("x", "y", "u", "v", "w", "z", "s", "a", "bb", "c")}
        t = T(v["y"]); K.axpby(T(v["a"]), T(v["x"]), T(v["bb"]), t)
        np.testing.assert_array_equal(t.cpu().numpy(), g[key + "_axpby"])
        t = T(v["y"]); K.add2_scaled(t, T(v["a"]), T(v["u"]), T(v["bb"]), T(v["v"]))
        np.testing.assert_array_equal(t.cpu().numpy(), g[key + "_add2"])
        d = K.dot_partial(T(v["x"]), T(v["y"])).cpu().numpy()
        np.testing.assert_allclose(d, g[key + "_dot"], rtol=1e-13, atol=1e-13)
        t = T(v["y"])
        d = K.fused_update_dot(T(v["a"]), T(v["x"]), T(v["bb"]), t).cpu().numpy()
        np.testing.assert_array_equal(t.cpu().numpy(), g[key + "_ud_y"])
        np.testing.assert_allclose(d, g[key + "_ud_dot"], rtol=1e-13)
        t1, t2 = T(v["y"]), T(v["w"])
        K.fused_paired_update(t1, T(v["a"]), T(v["u"]), T(v["bb"]), T(v["s"]), t2, T(v["c"]), T(v["x"]))
        np.testing.assert_array_equal(t1.cpu().numpy(), g[key + "_pu_y1"])
        np.testing.assert_array_equal(t2.cpu().numpy(), g[key + "_pu_y2"])
        t = T(v["y"])
        d1, d2 = K.fused_update_dot2(t, T(v["u"]), T(v["c"]), T(v["w"]), T(v["z"]))
        np.testing.assert_array_equal(t.cpu().numpy(), g[key + "_ud2_y"])
        np.testing.assert_allclose(d1.cpu().numpy(), g[key + "_ud2_d1"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(d2.cpu().numpy(), g[key + "_ud2_d2"], rtol=1e-13)


@pytest.mark.parametrize("n,m", [(0, 3), (1, 1), (7, 64), (1_000_003, 8), (300_001, 1)])
def test_dot_large_and_edges(n, m, rng):
    x = rng.standard_normal((n, m))
    y = rng.standard_normal((n, m))
    d = K.dot_partial(T(x), T(y)).cpu().numpy()
    ref = (x * y).sum(axis=0) if n else np.zeros(m)
    np.testing.assert_allclose(d, ref, rtol=1e-11, atol=1e-9)
    # deterministic: same bits on a rerun
    d2 = K.dot_partial(T(x), T(y)).cpu().numpy()
    np.testing.assert_array_equal(d, d2)


def test_scalar_broadcast_and_count_checks(rng):
    from paper_2103_07329_b200.errors import InvalidArgumentError, ShapeMismatchError
    x = T(rng.standard_normal((10, 4)))
    y = T(rng.standard_normal((10, 4)))
    ref = 2.0 * x.cpu().numpy() + 0.5 * y.cpu().numpy()
    K.axpby(2.0, x, 0.5, y)
    np.testing.assert_array_equal(y.cpu().numpy(), ref)
    with pytest.raises(InvalidArgumentError):
        K.axpby([1.0, 2.0], x, 1.0, y)
    with pytest.raises(ShapeMismatchError):
        K.axpby(1.0, T(np.zeros((9, 4))), 1.0, y)


@pytest.mark.parametrize("m", [1, 4, 8, 16])
def test_slab_compressed_indices_bitwise(m, rng):
    """Slab-relative 16-bit columns (2 B/nnz less) give the same bits as the
    32-bit columns and as the oracle."""
    from paper_2103_07329_b200.io import gen_random_sdd
    A = gen_random_sdd(n=150_000, band=4096, seed=5)
    D32 = K.DeviceCsr.from_block(A)
    D16 = K.DeviceCsr.from_block(A, slab=True)
    assert D16.col_idx.dtype == torch.uint16 and D16.slab_base is not None
    x = T(rng.standard_normal((A.ncols, m)))
    b = T(rng.standard_normal((A.nrows, m)))
    for mode in range(4):
        y0 = rng.standard_normal((A.nrows, m))
        y32, y16 = T(y0), T(y0)
        K.csr_spmv(D32, None, None, x, y32, mode, b)
        K.csr_spmv(D16, None, None, x, y16, mode, b)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y16.cpu().numpy(), y32.cpu().numpy())
    ref = np.empty((A.nrows, m))
    O.csr_spmv(A.row_ptr, A.col_idx, A.values, x.cpu().numpy(), ref, 0)
    y = torch.empty(A.nrows, m, dtype=torch.float64, device=DEV)
    K.csr_spmv(D16, None, None, x, y, 0)
    np.testing.assert_array_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("m", [1, 3, 8, 16])
@pytest.mark.parametrize("vdt", [np.float64, np.float32])
@pytest.mark.parametrize("width", [np.uint16, np.uint32])
@pytest.mark.parametrize("forward", [True, False])
def test_gs_sweep_vs_oracle_bitwise(m, vdt, width, forward, rng):
    """Level-scheduled Gauss-Seidel half-sweep == the sequential sweep
    (_ckernels.pyx:60-79) bitwise, on random NONSYMMETRIC patterns (rows that
    must still see an old value constrain the schedule too) with a nonzero
    off-leaf coupling c."""
    from mrs_testutil import random_csr
    n = 4000
    blk = random_csr(n, n, 9.0, rng, diag=8.0)
    ci = blk.col_idx.astype(width)
    v = blk.values.astype(vdt)
    dp = O.diag_positions(O.Csr(n, n, blk.row_ptr, blk.col_idx, blk.values))
    b = rng.standard_normal((n, m))
    c = rng.standard_normal((n, m))
    x0 = rng.standard_normal((n, m))
    ref = x0.copy()
    O.gs_sweep(blk.row_ptr, ci, v, dp, b, c, ref, forward)
    x = T(x0)
    K.gs_sweep(T(blk.row_ptr.astype(np.int32)), T(ci), T(v), T(dp), T(b), T(c), x, forward)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(x.cpu().numpy(), ref)


@pytest.mark.parametrize("m", [4, 16])
def test_gs_sweep_slab_indices_symmetric_pair(m, rng):
    """Forward + backward on a 7-point operator stored with slab-relative
    16-bit columns (as the solver uploads it) == the oracle.  ~330 rows per
    schedule level: m=4 runs the one-CTA kernel, m=16 the cluster kernel."""
    from paper_2103_07329_b200.io import gen_poisson3d
    A, _ = gen_poisson3d(20, 20, 180)          # 72k rows: slab-compressed columns
    D = K.DeviceCsr.from_block(A, slab=True)
    assert D.slab_base is not None
    dp = O.diag_positions(O.Csr.of(A))
    b = rng.standard_normal((A.nrows, m))
    zero = np.zeros_like(b)
    ref = np.zeros_like(b)
    x = T(ref)
    for fwd in (True, False):
        O.gs_sweep(A.row_ptr, A.col_idx, A.values, dp, b, zero, ref, fwd)
        K.gs_sweep(D, None, None, T(dp), T(b), T(zero), x, fwd)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(x.cpu().numpy(), ref)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("vdt", [np.float64, np.float32])
@pytest.mark.parametrize("slab", [False, True])
def test_spmv_long_rows_bitwise(m, vdt, slab, rng):
    """Rows far longer than the mean (the AMG coarse-level pattern) run on
    whole CTAs (kernels.long_row_split): still bitwise the reference order."""
    import scipy.sparse as sp
    n = 6000
    base = sp.random(n, n, density=8.0 / n, random_state=7, format="csr")
    rows, cols = [], []
    for i in rng.choice(n, 40, replace=False):
        L = int(rng.integers(300, 3000))             # > one 2048-product chunk at m = 1
        js = np.sort(rng.choice(n, L, replace=False))
        rows += [i] * L
        cols += list(js)
    M = (base + sp.csr_matrix((rng.standard_normal(len(rows)), (rows, cols)), shape=(n, n))).tocsr()
    M.sort_indices()
    blk = CsrBlock.from_scipy(M)
    vals = blk.values.astype(vdt)
    D = K.DeviceCsr(blk.row_ptr, blk.col_idx, vals, n, n, slab=slab)
    assert D.long_rows is not None and D.long_rows.numel() >= 40
    x = rng.standard_normal((n, m))
    b = rng.standard_normal((n, m))
    y0 = rng.standard_normal((n, m))
    for mode in range(4):
        y = T(y0)
        K.csr_spmv(D, None, None, T(x), y, mode, T(b) if mode == 3 else None)
        ref = y0.copy()
        O.csr_spmv(blk.row_ptr, blk.col_idx, vals, x, ref, mode, b if mode == 3 else None)
        np.testing.assert_array_equal(y.cpu().numpy(), ref, err_msg=f"mode {mode}")


@pytest.mark.parametrize("m", [4, 8, 16])
@pytest.mark.parametrize("vdt", [np.float64, np.float32])
@pytest.mark.parametrize("coop", [0, 1])
def test_spmv_coop_entry_loads_bitwise(m, vdt, coop, rng):
    """Operators with >= 12 entries per row (beyond the LONG range) load each
    entry once per lane group and shuffle it (spmm_coop): still bitwise."""
    from mrs_testutil import random_csr
    from paper_2103_07329_b200 import _lib
    n = 40000
    blk = random_csr(n, n, 20.0, rng)
    vals = blk.values.astype(vdt)
    x = rng.standard_normal((n, m))
    b = rng.standard_normal((n, m))
    y0 = rng.standard_normal((n, m))
    try:
        _lib.set_option("spmm_coop", coop)
        for mode in range(4):
            y = spmv_dev(blk.row_ptr, blk.col_idx, vals, x, y0, mode, b if mode == 3 else None)
            ref = y0.copy()
            O.csr_spmv(blk.row_ptr, blk.col_idx, vals, x, ref, mode, b if mode == 3 else None)
            np.testing.assert_array_equal(y, ref, err_msg=f"mode {mode}")
    finally:
        _lib.set_option("spmm_coop", 2)


@pytest.mark.parametrize("m", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("variant", [1, 2, 3, 4, 5, 7])
def test_every_spmm_variant_bitwise(m, variant, rng):
    """Every SpMM variant the per-operator choice can pick (lane, cooperative
    loads, 16 in flight, gathers through L2 only, L1::no_allocate) gives the
    reference kernel's bits, every mode, both value types, slab indices."""
    from mrs_testutil import random_csr
    from paper_2103_07329_b200 import _lib
    n = 20000
    blk = random_csr(n, n, 14.0, rng)
    x = rng.standard_normal((n, m))
    b = rng.standard_normal((n, m))
    y0 = rng.standard_normal((n, m))
    try:
        _lib.set_option("spmm_variant", variant)
        for vdt in (np.float64, np.float32):
            vals = blk.values.astype(vdt)
            for mode in range(4):
                y = spmv_dev(blk.row_ptr, blk.col_idx, vals, x, y0, mode, b if mode == 3 else None)
                ref = y0.copy()
                O.csr_spmv(blk.row_ptr, blk.col_idx, vals, x, ref, mode, b if mode == 3 else None)
                np.testing.assert_array_equal(y, ref, err_msg=f"variant {variant} mode {mode}")
    finally:
        _lib.set_option("spmm_variant", 0)


@pytest.mark.parametrize("m", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("vdt", [np.float64, np.float32])
def test_spmv_float32_vectors_bitwise(m, vdt, rng):
    """csr_spmv on float32 block vectors (extension): fp64 accumulation in entry
    order, ONE rounding at the store -- equal to the oracle kernel run on the
    widened operands and rounded once, every mode, plain and slab indices."""
    from mrs_testutil import random_csr
    n = 30000
    blk = random_csr(n, n, 11.0, rng)
    vals = blk.values.astype(vdt)
    x = rng.standard_normal((n, m)).astype(np.float32)
    b = rng.standard_normal((n, m)).astype(np.float32)
    y0 = rng.standard_normal((n, m)).astype(np.float32)
    for slab in (False, True):
        D = K.DeviceCsr(blk.row_ptr, blk.col_idx, vals, n, n, slab=slab)
        for mode in range(4):
            y = T(y0)
            K.csr_spmv(D, None, None, T(x), y, mode, T(b) if mode == 3 else None)
            ref = y0.astype(np.float64)
            O.csr_spmv(blk.row_ptr, blk.col_idx, vals, x.astype(np.float64), ref, mode,
                       b.astype(np.float64) if mode == 3 else None)
            np.testing.assert_array_equal(y.cpu().numpy(), ref.astype(np.float32),
                                          err_msg=f"mode {mode} slab {slab}")
    with pytest.raises(Exception):                       # mixed vector types are rejected
        K.csr_spmv(D, None, None, T(x), T(y0.astype(np.float64)), 0)
