"""AMG setup on the GPU: the Galerkin triple product
A_c = (R A) P of every level computed by csrc/spgemm.cu must reproduce the
host path (csrc/amg_setup.cpp, itself bitwise the reference's amg.setup, see
tests/test_setup_native.py) BIT FOR BIT: same structure, same values, every
level -- including scipy's unsorted intermediate R A, whose row order fixes the
summation order of the second product."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2103_07329_b200 import _lib, gen_poisson3d  # noqa: E402
from paper_2103_07329_b200.amg import AmgParams, setup  # noqa: E402
from paper_2103_07329_b200.io import gen_random_sdd, gen_stencil27_aniso  # noqa: E402


def build(A, params, mixed, gpu):
    _lib.set_option("setup_gpu", gpu)
    try:
        before = _lib.lib().mrs_galerkin_gpu_count()
        h = setup(A, params, mixed_precision=mixed)
        return h, _lib.lib().mrs_galerkin_gpu_count() - before
    finally:
        _lib.set_option("setup_gpu", 1)


CASES = {
    "poisson_24": (lambda: gen_poisson3d(24, 24, 24)[0], AmgParams(), False),
    "poisson_40_mixed": (lambda: gen_poisson3d(40, 40, 40)[0], AmgParams(), True),
    "poisson_30_aggressive": (lambda: gen_poisson3d(30, 30, 30)[0],
                              AmgParams(agg_num_levels=2, num_paths=2, coarse_matrix_size=500), False),
    "s27_28": (lambda: gen_stencil27_aniso(28, seed=4), AmgParams(), False),
    "random_sdd": (lambda: gen_random_sdd(n=60000, band=300), AmgParams(), False),
}


@pytest.mark.parametrize("case", list(CASES))
def test_gpu_galerkin_hierarchy_bitwise(case):
    mk, params, mixed = CASES[case]
    A = mk()
    h_host, n_host = build(A, params, mixed, 0)
    h_gpu, n_gpu = build(A, params, mixed, 1)
    assert n_host == 0
    assert n_gpu == h_gpu.nlevels - 1 and n_gpu >= 1
    assert h_gpu.nlevels == h_host.nlevels
    for l, (a, b) in enumerate(zip(h_host.levels, h_gpu.levels)):
        for name in ("A", "P", "R"):
            x, y = getattr(a, name), getattr(b, name)
            assert (x is None) == (y is None), (l, name)
            if x is None:
                continue
            assert (x.nrows, x.ncols) == (y.nrows, y.ncols), (l, name)
            np.testing.assert_array_equal(x.row_ptr, y.row_ptr, err_msg=f"level {l} {name} row_ptr")
            np.testing.assert_array_equal(x.col_idx, y.col_idx, err_msg=f"level {l} {name} col_idx")
            assert x.values.dtype == y.values.dtype
            assert np.array_equal(x.values.view(np.uint8), y.values.view(np.uint8)), \
                f"level {l} {name} values differ"


@pytest.mark.parametrize("case", ["poisson_48", "s27_44", "random_sdd_wide"])
def test_device_slab_compression_matches_host(case, monkeypatch):
    """Index compression at upload on the device (csrc/slab.cu) vs on the host
    (core.slab_compress): same shift / bases (the plans stream the same bytes)
    and bitwise the same solve."""
    from paper_2103_07329_b200 import BlockVector
    from paper_2103_07329_b200.params import tree
    from paper_2103_07329_b200 import solvers as S
    A = {"poisson_48": lambda: gen_poisson3d(48, 48, 48)[0],
         "s27_44": lambda: gen_stencil27_aniso(44, seed=4),
         "random_sdd_wide": lambda: gen_random_sdd(n=200000, band=40000)}[case]()
    roles = {"solver": {"method": "CG", "rel_tolerance": "1e-8", "max_iters": "60"},
             "preconditioner": {"method": "MultiGrid"},
             "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
             "post_smoother": {"method": "Jacobi", "weight": "0.8"}}
    B = np.random.default_rng(5).uniform(-1, 1, (A.nrows, 4))
    out = {}
    for dev in (True, False):
        monkeypatch.setattr(_lib, "SLAB_ON_DEVICE", dev)
        cs = S.prepare(tree(roles), A)
        X = BlockVector.zeros(A.nrows, 4)
        st = cs.run(BlockVector.from_array(B), X)
        out[dev] = (st.iterations, X.data.copy(), cs.plan_factory(4).iteration_bytes)
    assert out[True][0] == out[False][0]
    assert out[True][2] == out[False][2], "different index widths / slab counts"
    assert np.array_equal(out[True][1], out[False][1])
