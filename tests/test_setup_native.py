"""Native (C++) AMG setup and eigenvalue bounds vs the reference's own output
(tests/golden/hierarchies.npz, eig.npz, produced by oracle/gen_golden.py).
CPU only: the setup is host code."""

import numpy as np
import pytest

from mrs_testutil import load_golden
from paper_2103_07329_b200.amg import AmgParams, estimate_eig_bounds, setup
from paper_2103_07329_b200.core import CsrBlock
from paper_2103_07329_b200.io import gen_poisson3d


def _blk(g, pre):
    nr, nc = g[pre + "_shape"]
    return CsrBlock(int(nr), int(nc), g[pre + "_rp"], g[pre + "_ci"], g[pre + "_v"], validate=False)


@pytest.mark.parametrize("name", ["p7_12", "p7_16_mixed", "p7_9x7x5_c50", "p27_10", "p7_12_agg"])
def test_native_setup_bitwise(golden_hier, name):
    g = golden_hier
    A = _blk(g, f"{name}_A")
    th, agg, npth, cs, ml, mixed = g[f"{name}_params"]
    h = setup(A, AmgParams(float(th), int(agg), int(npth), int(cs), int(ml)), bool(mixed))
    assert h.nlevels == int(g[f"{name}_nlevels"])
    for l, lv in enumerate(h.levels):
        for tag in ("A", "P", "R"):
            blk = getattr(lv, tag)
            key = f"{name}_L{l}_{tag}"
            if blk is None:
                assert key + "_rp" not in g
                continue
            np.testing.assert_array_equal(blk.row_ptr, g[key + "_rp"], err_msg=key)
            np.testing.assert_array_equal(blk.col_idx, g[key + "_ci"], err_msg=key)
            assert blk.col_idx.dtype == g[key + "_ci"].dtype, key
            assert blk.values.dtype == g[key + "_v"].dtype, key
            np.testing.assert_array_equal(blk.values, g[key + "_v"], err_msg=key)


def test_native_eig_bounds_bitwise():
    g = load_golden("eig.npz")
    A, _ = gen_poisson3d(9, 8, 7)
    assert estimate_eig_bounds(A) == tuple(g["p7_987"])
    assert estimate_eig_bounds(A.with_precision(__import__(
        "paper_2103_07329_b200.core", fromlist=["PrecisionTag"]).PrecisionTag.REDUCED)) == tuple(g["p7_987_f32"])
    assert estimate_eig_bounds(CsrBlock.from_dense(np.eye(32))) == tuple(g["eye32"])


def test_native_setup_matches_oracle_on_larger_grid():
    """32^3: the native setup equals the oracle restatement (itself pinned)."""
    from oracle.amg_setup import setup as osetup
    from oracle.oracle import Csr
    A, _ = gen_poisson3d(24, 20, 18)
    h = setup(A)
    ho = osetup(Csr.of(A))
    assert h.nlevels == len(ho.levels)
    for lv, lo in zip(h.levels, ho.levels):
        np.testing.assert_array_equal(lv.A.values, lo.A.values)
        np.testing.assert_array_equal(lv.A.col_idx.astype(np.int64), lo.A.col_idx.astype(np.int64))
        if lv.P is not None:
            np.testing.assert_array_equal(lv.P.values, lo.P.values)
            np.testing.assert_array_equal(lv.R.values, lo.R.values)
