"""Seeded system generators for the BASELINE.json configurations.

* :func:`gen_poisson3d` -- restatement of the reference generator
  (/root/reference/pkg/src/mrsolve/io.py:152-179): 7-point stencil, diagonal
  6, -1 to each existing neighbour (Dirichlet by elimination), x-fastest
  lexicographic ordering, right-hand side A @ 1.  Configs 1-3.
* :func:`gen_stencil27_aniso` -- config 4 (builder-defined):
  27-point variable-coefficient anisotropic SPD M-matrix.
* :func:`gen_random_sdd` -- config 5 (builder-defined):
  banded random symmetric diagonally dominant matrix.
* :func:`seeded_rhs` -- ``default_rng(seed).uniform(-1, 1, (n, m))``.

All return :class:`~paper_2103_07329_b200.core.CsrBlock` (int64 row_ptr,
smallest column width, float64 values), like the reference's ``CsrBlock``.
"""

from __future__ import annotations

import numpy as np

from .core import CsrBlock, BlockVector
from .errors import InvalidArgumentError
# XAMGBIN1 system files and YAML run configurations (reference io.py:46-149,
# :205-283) live in sysfile.py; re-exported here under the reference's names
from .sysfile import (MAGIC, BenchmarkSpec, SystemSpec, parse_run_config,  # noqa: F401
                      read_system, write_system)

__all__ = ["gen_poisson3d", "gen_stencil27_aniso", "gen_random_sdd", "seeded_rhs",
           "MAGIC", "read_system", "write_system", "SystemSpec", "BenchmarkSpec",
           "parse_run_config"]


def _block(n, ncols, indptr, indices, data):
    return CsrBlock.from_arrays(n, ncols, indptr, indices, data)


def gen_poisson3d(nx: int, ny: int, nz: int):
    """7-point Poisson operator and manufactured RHS A @ 1 (io.py:152-179).

    Built directly in sorted CSR order: the neighbours of row i in ascending
    column order are -z, -y, -x, self, +x, +y, +z.
    """
    if nx < 1 or ny < 1 or nz < 1:
        raise InvalidArgumentError("grid dimensions must be >= 1")
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    ix = idx % nx
    iy = (idx // nx) % ny
    iz = idx // (nx * ny)
    offs = [(-nx * ny, iz > 0), (-nx, iy > 0), (-1, ix > 0), (0, None),
            (1, ix < nx - 1), (nx, iy < ny - 1), (nx * ny, iz < nz - 1)]
    mask = np.stack([np.ones(n, bool) if m is None else m for _, m in offs], axis=1)
    cols = idx[:, None] + np.array([o for o, _ in offs], dtype=np.int64)[None, :]
    vals = np.where(np.array([o for o, _ in offs]) == 0, 6.0, -1.0)[None, :].repeat(n, 0)
    counts = mask.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    A = _block(n, n, indptr, cols[mask], vals[mask])
    # rhs = A @ ones: sum of the row in entry order (scipy csr @ dense order)
    rhs = np.zeros(n)
    vm = np.where(mask, vals, 0.0)
    acc = np.zeros(n)
    for k in range(7):          # scipy's csr_matvec sums entries in order
        acc = np.where(mask[:, k], acc + vm[:, k], acc)
    rhs[:] = acc
    return A, BlockVector.from_array(rhs)


def gen_stencil27_aniso(g: int, seed: int = 4, zaniso: float = 100.0,
                        kmin: float = 1e-2, kmax: float = 1e2):
    """Config 4: 3D anisotropic variable-coefficient 27-point stencil.

    Per cell k = exp(U(ln kmin, ln kmax)) from ``default_rng(seed)``.
    Off-diagonal a_ij = -w*s*sqrt(k_i k_j), w = 1/(|dx|+|dy|+|dz|),
    s = zaniso for the pure-z offsets (0,0,+-1) and 1 otherwise; diagonal
    a_ii = sum_j |a_ij| + sum over missing (boundary) neighbours of w*s*k_i,
    i.e. Dirichlet by elimination.  SPD M-matrix, nnz = (3g-2)^3.
    Generated plane by plane to bound host memory at g = 256.
    """
    if g < 1:
        raise InvalidArgumentError("grid size must be >= 1")
    n = g ** 3
    rng = np.random.default_rng(seed)
    k = np.exp(rng.uniform(np.log(kmin), np.log(kmax), n))
    offs = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    nnz = (3 * g - 2) ** 3
    indptr = np.zeros(n + 1, dtype=np.int64)
    indices = np.empty(nnz, dtype=np.uint32 if n > 65536 else np.int64)
    data = np.empty(nnz, dtype=np.float64)
    plane = g * g
    p = np.arange(plane, dtype=np.int64)
    px, py = p % g, p // g
    pos = 0
    for z in range(g):
        rows = z * plane + p
        ki = k[rows]
        cols = np.empty((plane, 27), dtype=np.int64)
        vals = np.zeros((plane, 27))
        mask = np.zeros((plane, 27), dtype=bool)
        diag = np.zeros(plane)
        ci = offs.index((0, 0, 0))
        for o, (dx, dy, dz) in enumerate(offs):
            if (dx, dy, dz) == (0, 0, 0):
                mask[:, o] = True
                cols[:, o] = rows
                continue
            w = 1.0 / (abs(dx) + abs(dy) + abs(dz))
            s = zaniso if (dx == 0 and dy == 0) else 1.0
            ok = ((px + dx >= 0) & (px + dx < g) & (py + dy >= 0) & (py + dy < g)
                  & (z + dz >= 0) & (z + dz < g))
            j = rows + dx + dy * g + dz * plane
            jj = np.where(ok, j, rows)
            a = -w * s * np.sqrt(ki * k[jj])
            vals[:, o] = np.where(ok, a, 0.0)
            mask[:, o] = ok
            cols[:, o] = jj
            diag += np.where(ok, -a, w * s * ki)
        vals[:, ci] = diag
        cnt = mask.sum(axis=1)
        m = int(cnt.sum())
        indices[pos:pos + m] = cols[mask]
        data[pos:pos + m] = vals[mask]
        indptr[z * plane + 1:(z + 1) * plane + 1] = pos + np.cumsum(cnt)
        pos += m
    assert pos == nnz
    return _block(n, n, indptr, indices, data)


def gen_random_sdd(n: int = 1 << 22, mean_upper: float = 7.5, band: int = 4096,
                   seed: int = 5):
    """Config 5: random symmetric strictly diagonally dominant banded matrix.

    Row i draws k_i ~ Poisson(mean_upper) offsets d ~ U{1..band} (duplicates
    dropped, j = i + d < n), values N(0, 1); mirrored to the lower triangle
    (so off-diagonals per row ~ Poisson(2 * mean_upper)); diagonal
    sum_j |a_ij| + 1.
    """
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    kc = rng.poisson(mean_upper, n)
    rows = np.repeat(np.arange(n, dtype=np.int64), kc)
    d = rng.integers(1, band + 1, rows.size)
    cols = rows + d
    vals = rng.standard_normal(rows.size)
    keep = cols < n
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    key = rows * (band + 1) + (cols - rows)
    _, first = np.unique(key, return_index=True)
    rows, cols, vals = rows[first], cols[first], vals[first]
    upper = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    sym = (upper + upper.T).tocsr()
    diag = np.asarray(abs(sym).sum(axis=1)).ravel() + 1.0
    mat = (sym + sp.diags(diag)).tocsr()
    mat.sort_indices()
    return CsrBlock.from_scipy(mat)


def seeded_rhs(n: int, m: int, seed: int = 0) -> np.ndarray:
    """BASELINE.json RHS: default_rng(seed).uniform(-1, 1, (n, m))."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (n, m))
