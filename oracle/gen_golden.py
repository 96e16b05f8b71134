"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the reference
is importable (oracle/_ref built by oracle/build_ref.sh, or the read-only
source tree /root/reference/pkg/src).  The committed fixtures pin both the
oracle restatement (oracle/oracle.py, oracle/mrs_oracle.c) and the device
path, and travel to the GPU box where the reference does not exist.

    python oracle/gen_golden.py            # rewrites tests/golden/

Every fixture stores the seeded inputs next to the reference outputs, so
tests never need the reference at run time.
"""

from __future__ import annotations

import hashlib
import os
import sys

# the reference's LAPACK coarse solve (scipy lu_solve) on ONE thread: threaded
# getrs rounds differently, and the oracle replays the 1-thread order
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")


def import_reference():
    os.environ.setdefault("MRSOLVE_KERNELS", "cython")
    for cand in (os.path.join(HERE, "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "mrsolve")):
            sys.path.insert(0, cand)
            break
    import mrsolve  # noqa: F401
    return mrsolve


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def gen_kernels(ms, rng):
    """Plugin KATs: csr_spmv over widths x precisions x modes x m, plus the
    blocked vector kernels (kernels/__init__.py:27-41)."""
    K = ms.kernels
    from mrsolve.core import CsrBlock, IndexWidth, compress_indices
    out = {}
    cases = []
    for ci, (n, ncols, dens, m) in enumerate([(37, 29, 0.3, 1), (64, 200, 0.1, 2),
                                              (150, 150, 0.05, 4), (300, 1000, 0.01, 8),
                                              (97, 66000, 0.0005, 1), (40, 40, 0.5, 16),
                                              (33, 33, 0.2, 32), (20, 20, 0.0, 2)]):
        a = rng.standard_normal((n, ncols)) * (rng.random((n, ncols)) < dens)
        if ci == 4:  # empty rows interleaved
            a[::3] = 0.0
        blk = CsrBlock.from_dense(a)
        x = rng.standard_normal((ncols, m))
        b = rng.standard_normal((n, m))
        y0 = rng.standard_normal((n, m))
        out[f"spmv{ci}_x"], out[f"spmv{ci}_b"], out[f"spmv{ci}_y0"] = x, b, y0
        for width in (IndexWidth.W8, IndexWidth.W16, IndexWidth.W32):
            if blk.ncols > width.capacity:
                continue
            wb = compress_indices(blk, width)
            for vdt in (np.float64, np.float32):
                key = f"spmv{ci}_w{int(width)}_{np.dtype(vdt).name}"
                out[key + "_rp"] = wb.row_ptr
                out[key + "_ci"] = wb.col_idx
                out[key + "_v"] = wb.values.astype(vdt)
                for mode in range(4):
                    y = y0.copy()
                    K.csr_spmv(wb.row_ptr, wb.col_idx, wb.values.astype(vdt), x, y,
                               mode, b=b if mode == 3 else None)
                    out[f"{key}_out{mode}"] = y
                cases.append(key)
    out["spmv_cases"] = np.array(cases)
    # blocked vector kernels
    vcases = []
    for vi, (n, m) in enumerate([(1, 1), (257, 1), (1000, 2), (333, 4), (1031, 8),
                                 (300, 16), (129, 32), (50, 3)]):
        x, y, u, v, w, z, s = (rng.standard_normal((n, m)) for _ in range(7))
        a, bb, c = (rng.standard_normal(m) for _ in range(3))
        key = f"vec{vi}"
        for nm, arr in dict(x=x, y=y, u=u, v=v, w=w, z=z, s=s, a=a, bb=bb, c=c).items():
            out[f"{key}_{nm}"] = arr
        t = y.copy(); K.axpby(a, x, bb, t); out[key + "_axpby"] = t
        t = y.copy(); K.add2_scaled(t, a, u, bb, v); out[key + "_add2"] = t
        out[key + "_dot"] = K.dot_partial(x, y)
        t = y.copy(); out[key + "_ud_dot"] = K.fused_update_dot(a, x, bb, t)
        out[key + "_ud_y"] = t
        t1, t2 = y.copy(), w.copy()  # y2 output buffer distinct from w
        K.fused_paired_update(t1, a, u, bb, s, t2, c, x)
        out[key + "_pu_y1"], out[key + "_pu_y2"] = t1, t2
        t = y.copy()
        d1, d2 = K.fused_update_dot2(t, u, c, w, z)
        out[key + "_ud2_y"], out[key + "_ud2_d1"], out[key + "_ud2_d2"] = t, d1, d2
        vcases.append(key)
    out["vec_cases"] = np.array(vcases)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def tree(ms, roles):
    t = ms.ParamTree()
    for role, entries in roles.items():
        t.add_map(role, {k: str(v) for k, v in entries.items()})
    t.set_defaults()
    return t


SOLVE_CASES = {
    # name: (grid, m, seed, roles)  -- shrunken BASELINE.json configs 1-3
    "c1_jacobi_pcg": ((12, 12, 12), 4, 0, {
        "solver": {"method": "CG", "rel_tolerance": "1e-8"},
        "preconditioner": {"method": "Jacobi"}}),
    "c2_amg_pcg": ((16, 16, 16), 4, 0, {
        "solver": {"method": "CG", "rel_tolerance": "1e-8"},
        "preconditioner": {"method": "MultiGrid"},
        "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
        "post_smoother": {"method": "Jacobi", "weight": "0.8"}}),
    "c3_amg_bicgstab_mixed": ((16, 16, 16), 4, 0, {
        "solver": {"method": "BiCGStab", "rel_tolerance": "1e-8"},
        "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": "1"},
        "pre_smoother": {"method": "Chebyshev", "polynomial_order": "2"},
        "post_smoother": {"method": "Chebyshev", "polynomial_order": "2"}}),
    "c2_amg_pcg_20": ((20, 18, 16), 2, 7, {
        "solver": {"method": "CG", "rel_tolerance": "1e-10"},
        "preconditioner": {"method": "MultiGrid", "mg_coarse_matrix_size": "100"},
        "pre_smoother": {"method": "Jacobi", "weight": "0.8", "max_iters": "2"},
        "post_smoother": {"method": "Jacobi", "weight": "0.8"}}),
    "plain_bicgstab": ((10, 10, 10), 3, 1, {
        "solver": {"method": "BiCGStab", "rel_tolerance": "1e-9"}}),
    "plain_cg": ((10, 10, 10), 2, 2, {
        "solver": {"method": "CG", "rel_tolerance": "1e-9"}}),
    "c3_amg_bicgstab_full_cheb3": ((14, 14, 14), 2, 3, {
        "solver": {"method": "BiCGStab", "rel_tolerance": "1e-8"},
        "preconditioner": {"method": "MultiGrid"},
        "pre_smoother": {"method": "Chebyshev", "polynomial_order": "3"},
        "post_smoother": {"method": "Chebyshev", "polynomial_order": "1"}}),
    # reordered / pipelined BiCGStab
    "rbicgstab_amg": ((16, 16, 16), 4, 4, {
        "solver": {"method": "RBiCGStab", "rel_tolerance": "1e-8"},
        "preconditioner": {"method": "MultiGrid"},
        "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
        "post_smoother": {"method": "Jacobi", "weight": "0.8"}}),
    "rbicgstab_plain_merged": ((10, 10, 10), 3, 5, {
        "solver": {"method": "RBiCGStab", "rel_tolerance": "1e-9", "merged": "1"}}),
    "pbicgstab_plain": ((10, 10, 10), 3, 6, {
        "solver": {"method": "PBiCGStab", "rel_tolerance": "1e-9"}}),
    "pbicgstab_amg_agg_cheb": ((16, 16, 16), 2, 7, {
        "solver": {"method": "PBiCGStab", "rel_tolerance": "1e-8", "max_iters": "20"},
        "preconditioner": {"method": "MultiGrid", "mg_agg_num_levels": "2",
                           "mg_coarse_matrix_size": "500", "mg_num_paths": "2"},
        "pre_smoother": {"method": "Chebyshev", "polynomial_order": "2"},
        "post_smoother": {"method": "Chebyshev", "polynomial_order": "2"}}),
    "pbicgstab_jacobi_merged": ((12, 12, 12), 2, 8, {
        "solver": {"method": "PBiCGStab", "rel_tolerance": "1e-8", "merged": "1"},
        "preconditioner": {"method": "Jacobi"}}),
    # hybrid Gauss-Seidel: the reference's DEFAULT
    # MultiGrid smoother, explicit directions / sweeps, and a GS preconditioner
    "amg_pcg_default_sgs": ((12, 12, 12), 2, 9, {
        "solver": {"method": "CG", "rel_tolerance": "1e-8"},
        "preconditioner": {"method": "MultiGrid"}}),
    "amg_bicgstab_gs_mixed": ((12, 10, 8), 3, 10, {
        "solver": {"method": "BiCGStab", "rel_tolerance": "1e-8"},
        "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": "1",
                           "mg_coarse_matrix_size": "60"},
        "pre_smoother": {"method": "Gauss-Seidel", "direction": "forward", "max_iters": "2"},
        "post_smoother": {"method": "Gauss-Seidel", "direction": "backward"}}),
    "sgs_precond_cg": ((10, 10, 10), 2, 11, {
        "solver": {"method": "CG", "rel_tolerance": "1e-9"},
        "preconditioner": {"method": "Gauss-Seidel"}}),
    # the other solver families of prepare (solvers.py:891-953) and the
    # Chebyshev preconditioner (:796-802)
    "mg_solver_jacobi": ((12, 12, 12), 2, 12, {
        "solver": {"method": "MultiGrid", "rel_tolerance": "1e-8", "max_iters": "60"},
        "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
        "post_smoother": {"method": "Jacobi", "weight": "0.8"}}),
    "mg_solver_default_sgs": ((10, 10, 10), 2, 13, {
        "solver": {"method": "MultiGrid", "rel_tolerance": "1e-8", "max_iters": "40",
                   "mg_coarse_matrix_size": "100"}}),
    "jacobi_solver": ((6, 6, 6), 2, 14, {
        "solver": {"method": "Jacobi", "rel_tolerance": "1e-4", "max_iters": "400",
                   "weight": "0.9"}}),
    "gs_solver": ((8, 8, 8), 3, 15, {
        "solver": {"method": "Gauss-Seidel", "rel_tolerance": "1e-6", "max_iters": "300"}}),
    "gs_solver_forward": ((6, 6, 6), 2, 16, {
        "solver": {"method": "Gauss-Seidel", "rel_tolerance": "1e-6", "max_iters": "300",
                   "direction": "forward"}}),
    "direct": ((6, 6, 6), 3, 17, {
        "solver": {"method": "Direct"}}),
    "cheb_precond_cg": ((12, 12, 12), 2, 18, {
        "solver": {"method": "CG", "rel_tolerance": "1e-9"},
        "preconditioner": {"method": "Chebyshev", "polynomial_order": "3"}}),
    "cheb_precond_bicgstab": ((10, 10, 10), 2, 19, {
        "solver": {"method": "BiCGStab", "rel_tolerance": "1e-9"},
        "preconditioner": {"method": "Chebyshev", "polynomial_order": "2"}}),
}


def gen_solves(ms):
    from mrsolve.core import BlockVector
    from mrsolve.io import gen_poisson3d
    out = {}
    for name, (grid, m, seed, roles) in SOLVE_CASES.items():
        A, _ = gen_poisson3d(*grid)
        n = A.nrows
        B = np.random.default_rng(seed).uniform(-1.0, 1.0, (n, m))
        cfg = tree(ms, roles)
        cs = ms.prepare(cfg, A)
        X = BlockVector.zeros(n, m)
        st = cs.run(BlockVector.from_array(B), X)
        out[f"{name}_B"] = B
        out[f"{name}_X"] = X.data
        out[f"{name}_iters"] = np.int64(st.iterations)
        out[f"{name}_rel"] = st.final_rel_residual
        out[f"{name}_hist"] = np.array(st.residual_history)
        h = cs.hierarchy
        if h is not None:
            out[f"{name}_nlevels"] = np.int64(h.nlevels)
            for l, lv in enumerate(h.levels):
                Ag = lv.A.blocks[0].diag   # 1x1 topology: stored precision
                out[f"{name}_L{l}_A_shape"] = np.array([Ag.nrows, Ag.nnz])
                out[f"{name}_L{l}_eig"] = np.array(lv.eig_bounds if lv.eig_bounds
                                                   else [np.nan, np.nan])
                for tag, blk in (("A", Ag), ("P", lv.P), ("R", lv.R)):
                    if blk is None:
                        continue
                    out[f"{name}_L{l}_{tag}_sha"] = np.array(
                        [sha(blk.row_ptr), sha(blk.col_idx.astype(np.int64)),
                         sha(blk.values)])
                    out[f"{name}_L{l}_{tag}_dtype"] = np.array(str(blk.values.dtype))
        print(f"{name}: n={n} m={m} iters={st.iterations} "
              f"levels={h.nlevels if h is not None else '-'} "
              f"maxrel={st.final_rel_residual.max():.3e}")
    out["solve_cases"] = np.array(list(SOLVE_CASES))
    np.savez_compressed(os.path.join(OUT, "solves.npz"), **out)


def gen_hierarchies(ms):
    """Full level arrays for small problems: the AMG-setup upload contract
    (amg.py:199-308), used to pin the native setup restatement bitwise."""
    from mrsolve.amg import AmgParams, setup
    from mrsolve.io import gen_poisson3d
    sys.path.insert(0, ROOT)
    from paper_2103_07329_b200.io import gen_stencil27_aniso
    out = {}
    probs = {
        "p7_12": (gen_poisson3d(12, 12, 12)[0], AmgParams(), False),
        "p7_16_mixed": (gen_poisson3d(16, 16, 16)[0], AmgParams(), True),
        "p7_9x7x5_c50": (gen_poisson3d(9, 7, 5)[0], AmgParams(coarse_matrix_size=50), False),
        "p27_10": (gen_stencil27_aniso(10, seed=4), AmgParams(), False),
        "p7_12_agg": (gen_poisson3d(12, 12, 12)[0],
                      AmgParams(agg_num_levels=1, num_paths=2), False),
    }
    for name, (A, prm, mixed) in probs.items():
        h = setup(A, prm, mixed_precision=mixed)
        out[f"{name}_nlevels"] = np.int64(h.nlevels)
        for l, lv in enumerate(h.levels):
            for tag, blk in (("A", lv.A.blocks[0].diag), ("P", lv.P), ("R", lv.R)):
                if blk is None:
                    continue
                out[f"{name}_L{l}_{tag}_rp"] = blk.row_ptr
                out[f"{name}_L{l}_{tag}_ci"] = blk.col_idx
                out[f"{name}_L{l}_{tag}_v"] = blk.values
                out[f"{name}_L{l}_{tag}_shape"] = np.array([blk.nrows, blk.ncols])
        out[f"{name}_A_rp"] = A.row_ptr
        out[f"{name}_A_ci"] = A.col_idx
        out[f"{name}_A_v"] = A.values
        out[f"{name}_A_shape"] = np.array([A.nrows, A.ncols])
        out[f"{name}_params"] = np.array([prm.strength_threshold, prm.agg_num_levels,
                                          prm.num_paths, prm.coarse_matrix_size,
                                          prm.max_levels, float(mixed)])
        print(f"{name}: levels={h.nlevels} rows={[lv.nrows for lv in h.levels]}")
    out["hier_cases"] = np.array(list(probs))
    np.savez_compressed(os.path.join(OUT, "hierarchies.npz"), **out)


def gen_generators(ms):
    from mrsolve.io import gen_poisson3d
    out = {}
    for dims in ((2, 1, 1), (3, 4, 5), (8, 8, 8)):
        A, b = gen_poisson3d(*dims)
        key = "poisson_%dx%dx%d" % dims
        out[key + "_rp"], out[key + "_ci"], out[key + "_v"] = A.row_ptr, A.col_idx, A.values
        out[key + "_b"] = b.data
    np.savez_compressed(os.path.join(OUT, "generators.npz"), **out)


def gen_eig(ms):
    from mrsolve.core import CsrBlock, SegmentedMatrix
    from mrsolve.io import gen_poisson3d
    from mrsolve.solvers import estimate_eig_bounds
    out = {}
    A, _ = gen_poisson3d(9, 8, 7)
    out["p7_987"] = np.array(estimate_eig_bounds(SegmentedMatrix.from_global(A)))
    A32 = A.with_precision(ms.PrecisionTag.REDUCED)
    out["p7_987_f32"] = np.array(estimate_eig_bounds(SegmentedMatrix.from_global(A32)))
    out["eye32"] = np.array(estimate_eig_bounds(
        SegmentedMatrix.from_global(CsrBlock.from_dense(np.eye(32)))))
    np.savez_compressed(os.path.join(OUT, "eig.npz"), **out)


def gen_sysfile(ms):
    """An XAMGBIN1 file written by the reference's own write_system
    (io.py:46-68): pins our reader and writer byte for byte."""
    from mrsolve.core import BlockVector
    from mrsolve.io import gen_poisson3d, write_system
    A, _ = gen_poisson3d(3, 2, 2)
    rng = np.random.default_rng(41)
    rhs = BlockVector.from_array(rng.standard_normal((A.nrows, 3)))
    guess = BlockVector.from_array(rng.standard_normal((A.nrows, 3)))
    write_system(os.path.join(OUT, "xamgbin1_ref.bin"), A, rhs, guess)


_JAC08 = {"method": "Jacobi", "weight": "0.8"}
_CHEB2 = {"method": "Chebyshev", "polynomial_order": "2"}
#: BASELINE.json configs at their FULL sizes (C1-C3 on the reference generator)
#: and the builder-defined C4 operator family (27-pt anisotropic) at sizes the
#: reference finishes in minutes: (kind, grid, m, seed, roles)
FULL_CASES = {
    "c1": ("p7", 32, 4, 0, {"solver": {"method": "CG", "rel_tolerance": "1e-8",
                                       "max_iters": "1000"},
                            "preconditioner": {"method": "Jacobi"}}),
    "c2": ("p7", 64, 8, 0, {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
                            "preconditioner": {"method": "MultiGrid"},
                            "pre_smoother": _JAC08, "post_smoother": _JAC08}),
    "c3": ("p7", 128, 16, 0, {"solver": {"method": "BiCGStab", "rel_tolerance": "1e-8"},
                              "preconditioner": {"method": "MultiGrid",
                                                 "mg_mixed_precision": "1"},
                              "pre_smoother": _CHEB2, "post_smoother": _CHEB2}),
    "c4_24": ("s27", 24, 8, 0, {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
                                "preconditioner": {"method": "MultiGrid"},
                                "pre_smoother": _JAC08, "post_smoother": _JAC08}),
    "c4_32": ("s27", 32, 8, 0, {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
                                "preconditioner": {"method": "MultiGrid"},
                                "pre_smoother": _JAC08, "post_smoother": _JAC08}),
    "c4_64": ("s27", 64, 8, 0, {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
                                "preconditioner": {"method": "MultiGrid"},
                                "pre_smoother": _JAC08, "post_smoother": _JAC08}),
    "c4_128": ("s27", 128, 8, 0, {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
                                  "preconditioner": {"method": "MultiGrid"},
                                  "pre_smoother": _JAC08, "post_smoother": _JAC08}),
    # BASELINE.json config 4 at its full size (449 M nnz; ~30 min, ~40 GB)
    "c4_256": ("s27", 256, 8, 0, {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
                                  "preconditioner": {"method": "MultiGrid"},
                                  "pre_smoother": _JAC08, "post_smoother": _JAC08}),
}
#: rows of X stored per case (strided sample; the full X hash is stored too)
SAMPLE_ROWS = 4096


def sample_rows(n: int) -> np.ndarray:
    """Strided row sample of an n-row solution (first and last row included)."""
    if n <= SAMPLE_ROWS:
        return np.arange(n)
    return np.unique(np.concatenate([np.linspace(0, n - 1, SAMPLE_ROWS).astype(np.int64),
                                     [n - 1]]))


def gen_fullsize(ms, names=None):
    """Reference outputs at BASELINE.json's full sizes (C1-C3) and for the C4
    operator family: iterations, residual history, final relative residuals,
    a strided X sample + the full-X hash, and per-level (rows, nnz, SHA) of
    the reference hierarchy with its Chebyshev eigenvalue bounds.  One file
    per case (tests/golden/full_<case>.npz) so cases can be regenerated alone.
    C3 takes ~3 min and c4_64 a few minutes on one core."""
    import time
    from mrsolve.core import BlockVector, CsrBlock
    from mrsolve.io import gen_poisson3d
    sys.path.insert(0, ROOT)
    from paper_2103_07329_b200.io import gen_stencil27_aniso
    for name, (kind, g, m, seed, roles) in FULL_CASES.items():
        if names and name not in names:
            continue
        if kind == "p7":
            A, _ = gen_poisson3d(g, g, g)
        else:
            G = gen_stencil27_aniso(g, seed=4)
            A = CsrBlock(G.nrows, G.ncols, G.row_ptr, G.col_idx, G.values)
        n = A.nrows
        B = np.random.default_rng(seed).uniform(-1.0, 1.0, (n, m))
        t0 = time.perf_counter()
        cs = ms.prepare(tree(ms, roles), A)
        t_setup = time.perf_counter() - t0
        X = BlockVector.zeros(n, m)
        t0 = time.perf_counter()
        st = cs.run(BlockVector.from_array(B), X)
        t_solve = time.perf_counter() - t0
        rows = sample_rows(n)
        out = {"kind": np.array(kind), "grid": np.int64(g), "m": np.int64(m),
               "seed": np.int64(seed), "iters": np.int64(st.iterations),
               "rel": st.final_rel_residual, "hist": np.array(st.residual_history),
               "rows": rows, "X_rows": X.data[rows], "X_sha": np.array(sha(X.data)),
               "X_norm": np.linalg.norm(X.data, axis=0), "B_sha": np.array(sha(B)),
               "t_setup": np.float64(t_setup), "t_solve": np.float64(t_solve)}
        h = cs.hierarchy
        if h is not None:
            out["nlevels"] = np.int64(h.nlevels)
            for l, lv in enumerate(h.levels):
                Ag = lv.A.blocks[0].diag
                out[f"L{l}_A_shape"] = np.array([Ag.nrows, Ag.nnz])
                out[f"L{l}_eig"] = np.array(lv.eig_bounds if lv.eig_bounds else [np.nan, np.nan])
                for tag, blk in (("A", Ag), ("P", lv.P), ("R", lv.R)):
                    if blk is None:
                        continue
                    out[f"L{l}_{tag}_sha"] = np.array(
                        [sha(blk.row_ptr.astype(np.int64)), sha(blk.col_idx.astype(np.int64)),
                         sha(blk.values)])
                    out[f"L{l}_{tag}_dtype"] = np.array(str(blk.values.dtype))
        np.savez_compressed(os.path.join(OUT, f"full_{name}.npz"), **out)
        print(f"full {name}: n={n} m={m} iters={st.iterations} "
              f"levels={h.nlevels if h is not None else '-'} "
              f"maxrel={st.final_rel_residual.max():.3e} setup {t_setup:.1f}s "
              f"solve {t_solve:.1f}s", flush=True)


def main():
    """All fixtures, or only the named groups (e.g. ``gen_golden.py solves``;
    ``gen_golden.py fullsize[:c2,c4_24]`` for the full-size reference runs)."""
    args = sys.argv[1:]
    full = [a for a in args if a.startswith("fullsize")]
    if full:
        ms = import_reference()
        assert ms.kernels.BACKEND == "cython", ms.kernels.BACKEND
        os.makedirs(OUT, exist_ok=True)
        sel = full[0].split(":", 1)[1].split(",") if ":" in full[0] else None
        gen_fullsize(ms, sel)
        return
    ms = import_reference()
    assert ms.kernels.BACKEND == "cython", ms.kernels.BACKEND
    os.makedirs(OUT, exist_ok=True)
    want = set(sys.argv[1:]) or {"kernels", "generators", "eig", "solves", "hierarchies",
                                 "sysfile"}
    if "kernels" in want:
        gen_kernels(ms, np.random.default_rng(20240817))
    if "generators" in want:
        gen_generators(ms)
    if "eig" in want:
        gen_eig(ms)
    if "solves" in want:
        gen_solves(ms)
    if "hierarchies" in want:
        gen_hierarchies(ms)
    if "sysfile" in want:
        gen_sysfile(ms)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
