"""The hierarchies the full-size solves upload, pinned to the reference's own.

tests/golden/full_<case>.npz hold, per level of the hierarchy the reference's
``amg.setup`` built for BASELINE.json's C2 (64^3) and C3 (128^3, mixed
precision) systems and for the C4 operator family (27-point anisotropic,
24^3 .. 128^3), the SHA-256 of (row_ptr, col_idx, values) of A, P and R plus
the Chebyshev eigenvalue bounds (oracle/gen_golden.py ``fullsize``).  The
native setup (csrc/amg_setup.cpp) must reproduce every array bitwise -- the
device solves of tests/test_gpu_fullsize.py then run on the reference's
hierarchy.  CPU only.
"""

import hashlib
import os

import numpy as np
import pytest

from mrs_testutil import GOLDEN, load_golden
from paper_2103_07329_b200.amg import AmgParams, estimate_eig_bounds, setup
from paper_2103_07329_b200.io import gen_poisson3d, gen_stencil27_aniso

CASES = [c for c in ("c2", "c3", "c4_24", "c4_32", "c4_64", "c4_128")
         if os.path.exists(os.path.join(GOLDEN, f"full_{c}.npz"))]


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def _matrix(g):
    grid = int(g["grid"])
    if str(g["kind"]) == "p7":
        return gen_poisson3d(grid, grid, grid)[0]
    return gen_stencil27_aniso(grid, seed=4)


@pytest.mark.parametrize("case", CASES)
def test_native_hierarchy_equals_reference(case):
    g = load_golden(f"full_{case}.npz")
    mixed = case == "c3"
    h = setup(_matrix(g), AmgParams(), mixed_precision=mixed)
    assert h.nlevels == int(g["nlevels"])
    for l, lv in enumerate(h.levels):
        assert [lv.A.nrows, lv.A.nnz] == list(g[f"L{l}_A_shape"]), (case, l)
        for tag in ("A", "P", "R"):
            blk = getattr(lv, tag)
            key = f"L{l}_{tag}_sha"
            if blk is None:
                assert key not in g.files, (case, l, tag)
                continue
            got = [_sha(blk.row_ptr.astype(np.int64)), _sha(blk.col_idx.astype(np.int64)),
                   _sha(blk.values)]
            assert got == list(g[key]), (case, l, tag)
            assert str(blk.values.dtype) == str(g[f"L{l}_{tag}_dtype"]), (case, l, tag)


@pytest.mark.skipif("c3" not in CASES, reason="full_c3.npz not generated")
def test_native_eig_bounds_equal_reference_c3():
    """C3's Chebyshev bounds (power iteration per level, solvers.py:486-517)."""
    g = load_golden("full_c3.npz")
    h = setup(_matrix(g), AmgParams(), mixed_precision=True)
    for l, lv in enumerate(h.levels[:-1]):
        assert estimate_eig_bounds(lv.A) == tuple(g[f"L{l}_eig"]), l


def _oracle_full(case):
    """Re-run a full-size golden case through the CPU oracle (1x1 topology:
    the oracle replays the reference arithmetic exactly)."""
    import hashlib as _h
    from oracle import oracle as O
    from oracle.amg_setup import setup as osetup
    g = load_golden(f"full_{case}.npz")
    A = O.Csr.of(_matrix(g))
    m = int(g["m"])
    B = np.random.default_rng(int(g["seed"])).uniform(-1.0, 1.0, (A.nrows, m))
    assert _sha(B) == str(g["B_sha"])
    X = np.zeros_like(B)
    if case == "c1":
        st = O.cg_solve(A, B, X, O.JacobiPrecond(A, 1.0, 1), 1e-8, 1000)
    else:
        mg = O.MultiGrid(osetup(A), ("jacobi", 0.8, 1), ("jacobi", 0.8, 1))
        st = O.cg_solve(A, B, X, mg, 1e-8, 100)
    return g, st, X


@pytest.mark.parametrize("case", [c for c in ("c1", "c4_24") if
                                  os.path.exists(os.path.join(GOLDEN, f"full_{c}.npz"))])
def test_oracle_reproduces_full_size_reference(case):
    g, st, X = _oracle_full(case)
    assert st.iterations == int(g["iters"])
    assert _sha(X) == str(g["X_sha"])
    np.testing.assert_array_equal(np.array(st.residual_history), g["hist"])
    np.testing.assert_array_equal(st.final_rel_residual, g["rel"])
