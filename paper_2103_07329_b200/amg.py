"""AMG hierarchy: the reference's Ruge-Stueben setup, run natively.

The solve phase consumes the hierarchy the reference's ``amg.setup``
(/root/reference/pkg/src/mrsolve/amg.py:254-308) produces.  :func:`setup`
computes exactly that hierarchy -- bitwise, pinned by
tests/test_setup_native.py against tests/golden/hierarchies.npz -- in C++
(csrc/amg_setup.cpp) instead of Python loops, and returns the reference's
data model (:class:`Level`, :class:`Hierarchy`, amg.py:199-239).  A
hierarchy built by the reference itself is accepted too (duck-typed).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import CsrBlock, PrecisionTag, as_csr, choose_width
from .errors import InvalidArgumentError, SingularDiagonalError

__all__ = ["AmgParams", "Level", "Hierarchy", "setup", "estimate_eig_bounds", "coarse_inverse",
           "vcycle_tail_operator", "dense_tail_level", "set_dense_tail_rows"]


@dataclass(frozen=True)
class AmgParams:
    """amg.py:34-52 (same defaults and validation)."""

    strength_threshold: float = 0.25
    agg_num_levels: int = 0
    num_paths: int = 1
    coarse_matrix_size: int = 500
    max_levels: int = 25
    stall_ratio: float = 0.9

    def __post_init__(self):
        if not (0.0 < self.strength_threshold < 1.0):
            raise InvalidArgumentError("strength_threshold must be in (0, 1)")
        if self.coarse_matrix_size < 1:
            raise InvalidArgumentError("coarse_matrix_size must be >= 1")
        if self.max_levels < 2:
            raise InvalidArgumentError("max_levels must be >= 2")
        if self.num_paths < 1:
            raise InvalidArgumentError("num_paths must be >= 1")


@dataclass
class Level:
    """One level: operator, transfer pair, smoother state (amg.py:199-212)."""

    A: CsrBlock
    precision: PrecisionTag = PrecisionTag.FULL
    P: CsrBlock | None = None
    R: CsrBlock | None = None
    eig_bounds: tuple | None = None
    lu: object = None            # coarsest level: dense inverse (device solve)

    @property
    def nrows(self) -> int:
        return self.A.nrows


@dataclass
class Hierarchy:
    levels: list = field(default_factory=list)
    params: AmgParams | None = None
    mixed_precision: bool = False

    @property
    def nlevels(self) -> int:
        return len(self.levels)

    @property
    def coarsest(self) -> Level:
        return self.levels[-1]

    def operator_complexity(self) -> float:
        return sum(lv.A.nnz for lv in self.levels) / self.levels[0].A.nnz

    def stats_report(self) -> str:
        lines = ["level        rows          nnz  precision"]
        for i, lv in enumerate(self.levels):
            lines.append(f"{i:>5} {lv.nrows:>11} {lv.A.nnz:>12}  {lv.precision.value}")
        lines.append(f"operator complexity: {self.operator_complexity():.3f}")
        return "\n".join(lines)

    @classmethod
    def of(cls, h) -> "Hierarchy":
        """Adopt a reference ``mrsolve.amg.Hierarchy`` (1x1 topology)."""
        if isinstance(h, Hierarchy):
            return h
        out = []
        for lv in h.levels:
            A = lv.A
            if hasattr(A, "blocks") and len(A.blocks) == 1:
                A = A.blocks[0].diag          # stored precision of the level
            out.append(Level(as_csr(A), PrecisionTag(lv.precision.value),
                             as_csr(lv.P) if lv.P is not None else None,
                             as_csr(lv.R) if lv.R is not None else None,
                             lv.eig_bounds))
        return cls(out, getattr(h, "params", None), getattr(h, "mixed_precision", False))


def _copy_out(hc: _lib.mrs_host_csr) -> CsrBlock:
    n, nnz = hc.nrows, hc.nnz
    rp = np.ctypeslib.as_array(C.cast(hc.row_ptr, C.POINTER(C.c_int64)), (n + 1,)).copy()
    ci = np.ctypeslib.as_array(C.cast(hc.col_idx, C.POINTER(C.c_uint32)), (max(nnz, 1),))[:nnz]
    if hc.val_bytes == 8:
        v = np.ctypeslib.as_array(C.cast(hc.values, C.POINTER(C.c_double)), (max(nnz, 1),))[:nnz].copy()
    else:
        v = np.ctypeslib.as_array(C.cast(hc.values, C.POINTER(C.c_float)), (max(nnz, 1),))[:nnz].copy()
    width = choose_width(max(int(hc.ncols), 1))
    return CsrBlock(n, hc.ncols, rp, ci.astype(width.dtype), v, validate=False)


def setup(A_fine, params: AmgParams | None = None, mixed_precision: bool = False,
          topology=None) -> Hierarchy:
    """Build the level hierarchy of ``A_fine`` (reference amg.setup)."""
    A = as_csr(A_fine)
    if A.nrows != A.ncols:
        raise InvalidArgumentError("AMG setup requires a square matrix")
    params = params or AmgParams()
    keep: list = []
    hc = _lib.host_csr(A, keep)
    prm = _lib.mrs_amg_params(params.strength_threshold, params.agg_num_levels,
                              params.num_paths, params.coarse_matrix_size, params.max_levels,
                              params.stall_ratio, int(bool(mixed_precision)))
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.mrs_amg_setup(C.byref(hc), C.byref(prm), C.byref(h)), "AMG setup")
    try:
        levels = []
        for l in range(L.mrs_hier_nlevels(h)):
            out = {}
            for which, tag in ((0, "A"), (1, "P"), (2, "R")):
                hcsr = _lib.mrs_host_csr()
                if L.mrs_hier_get(h, l, which, C.byref(hcsr)) == 0:
                    out[tag] = _copy_out(hcsr)
            prec = PrecisionTag.REDUCED if (mixed_precision and l > 0) else PrecisionTag.FULL
            levels.append(Level(out["A"], prec, out.get("P"), out.get("R")))
    finally:
        L.mrs_hier_destroy(h)
    return Hierarchy(levels, params, bool(mixed_precision))


def estimate_eig_bounds(A, iterations: int = 10, seed: int = 12345) -> tuple[float, float]:
    """Power-iteration bounds of D^-1 A (solvers.py:486-517), native; the start
    vector is numpy's ``default_rng(seed).standard_normal(n)`` as in the
    reference."""
    A = as_csr(A)
    d = A.diagonal()
    if np.any(d == 0.0):
        raise SingularDiagonalError("eigenvalue estimation needs a nonzero diagonal")
    start = np.ascontiguousarray(np.random.default_rng(seed).standard_normal(A.nrows))
    keep: list = []
    hc = _lib.host_csr(A, keep)
    lo, hi = C.c_double(), C.c_double()
    _lib.check(_lib.lib().mrs_eig_bounds(C.byref(hc), iterations, 0, start.ctypes.data,
                                         C.byref(lo), C.byref(hi)), "eigenvalue bounds")
    return (lo.value, hi.value)


def coarse_inverse(A) -> np.ndarray:
    """Dense inverse of the coarsest operator for the device coarse solve
    (replaces the cached LU of solvers.py:578-585 / :644-649)."""
    import scipy.linalg
    from .errors import SingularMatrixError
    A = as_csr(A)
    dense = A.to_dense().astype(np.float64)
    lu, piv = scipy.linalg.lu_factor(dense, check_finite=False)
    udiag = np.abs(np.diag(lu))
    scale = max(np.abs(dense).max(), 1.0) if dense.size else 1.0
    if udiag.size and udiag.min() <= 1e-14 * scale:
        raise SingularMatrixError("matrix is singular to working precision")
    return np.ascontiguousarray(scipy.linalg.lu_solve((lu, piv), np.eye(A.nrows), check_finite=False))


#: Largest level (rows) the V-cycle tail may be collapsed from (dense n x n
#: operator, n^2 * 8 bytes); 0 disables.  Env MRS_DENSE_TAIL_ROWS.
DENSE_TAIL_ROWS = int(os.environ.get("MRS_DENSE_TAIL_ROWS", "8000"))
# cost model of the choice (microseconds; B200 measurements, profiles/r01_ab_experiments.txt):
# a solve-path kernel costs ~_T_LAUNCH plus _T_ROUND per dependent load round of its
# longest row (16 entries in flight); the dense product streams n^2*8 bytes at _DENSE_BW
_T_LAUNCH, _T_ROUND = 3.0, 1.0                           # us, us
_DENSE_BW = float(os.environ.get("MRS_DENSE_BW", "3e6"))     # bytes/us (DMMA kernel)
_SGS_KERNEL_FACTOR = 10     # a Gauss-Seidel half-sweep ~ 10 SpMM launches (schedule barriers)


def set_dense_tail_rows(n: int) -> None:
    """Row cap of the collapsed V-cycle tail (0: per-level kernels)."""
    global DENSE_TAIL_ROWS
    DENSE_TAIL_ROWS = max(0, int(n))


def _kernel_us(M) -> float:
    if M is None:
        return 0.0
    M = as_csr(M)
    longest = int(np.diff(M.row_ptr).max()) if M.nrows else 0
    return _T_LAUNCH + _T_ROUND * 2 * -(-longest // 16)


def dense_tail_level(levels, limit=None, pre=None, post=None) -> int:
    """Level l >= 1 (not the coarsest, at most ``limit`` rows) whose collapsed
    tail saves the most estimated time per V-cycle, or -1 (none saves).

    Saving of collapsing at l = the per-level kernels of levels l..L-2
    (smoother + residual sweeps over A_j, the two transfers) and the coarse
    solve, each ~ launch + dependent load rounds of its longest row;
    cost = streaming the dense n_l x n_l operator."""
    limit = DENSE_TAIL_ROWS if limit is None else limit
    if limit <= 0 or len(levels) < 3:
        return -1

    def a_kernels(sm):
        if sm is None:
            return 2
        if sm.kind == _lib.SMOOTH_CHEBYSHEV:
            return max(sm.order, 1)
        if sm.kind == _lib.SMOOTH_SGS:        # level-scheduled half-sweeps: one
            halves = 2 if sm.direction == 0 else 1      # barrier per schedule level
            return _SGS_KERNEL_FACTOR * halves * max(sm.sweeps, 1)
        return max(sm.sweeps, 1)
    ka = a_kernels(pre) + a_kernels(post)   # (zero-guess first step is fused: ~ +residual)
    nL = as_csr(levels[-1][0]).nrows
    saving = _T_LAUNCH + nL * nL * 8.0 / _DENSE_BW           # coarse solve
    best, best_gain = -1, 0.0
    for l in range(len(levels) - 2, 0, -1):
        A, P, R, _ = levels[l]
        saving += ka * _kernel_us(A) + _kernel_us(P) + _kernel_us(R)
        n = as_csr(A).nrows
        if n > limit:
            break
        gain = saving - (_T_LAUNCH + n * n * 8.0 / _DENSE_BW)
        if gain > best_gain:
            best, best_gain = l, gain
    return best


def vcycle_tail_operator(levels, start: int, pre, post, inv) -> np.ndarray | None:
    """Dense operator T of the V-cycle from level ``start`` down (setup phase).

    Below the fine levels a V-cycle entered with a zero guess is a fixed
    LINEAR map of its right-hand side: x_l = T_l b_l (the zero-guess
    pre-smoother, residual, restriction, the recursion, prolongation and
    post-smoother of solvers.py:651-664 are all linear in b_l).  T_l is built
    here once by applying that sub-V-cycle to the n_l unit vectors (fp64,
    values widened like the device kernels), so the solve runs the whole tail
    as one dense product -- one launch instead of ~4 per level.  Same operator
    as the per-level kernels; only the floating-point evaluation order of the
    tail differs (the reference's coarsest LU is replaced the same way, see
    coarse_inverse).  ``levels``: (A, P, R, eig_bounds) per level; pre/post:
    _lib.mrs_smoother.  Returns None for Gauss-Seidel smoothing (kept on the
    exact level-scheduled kernels).
    """
    for sm in (pre, post):
        if sm.kind not in (_lib.SMOOTH_JACOBI, _lib.SMOOTH_CHEBYSHEV, _lib.SMOOTH_SGS):
            return None
    mats = []
    for (A, P, R, bounds) in levels[start:]:
        A = as_csr(A)
        As = A.to_scipy()
        mats.append((As, A.diagonal().astype(np.float64),
                     as_csr(P).to_scipy() if P is not None else None,
                     as_csr(R).to_scipy() if R is not None else None, bounds))

    gs_rows = {}

    def gs_half(k, b, x, forward):            # _ckernels.pyx:60-79, in place on x
        if k not in gs_rows:
            As = mats[k][0]
            rows = []
            for i in range(As.shape[0]):
                lo, hi = As.indptr[i], As.indptr[i + 1]
                cols, vals = As.indices[lo:hi], As.data[lo:hi]
                off = cols != i
                rows.append((cols[off], vals[off], vals[~off][0]))
            gs_rows[k] = rows
        rows = gs_rows[k]
        order = range(len(rows)) if forward else range(len(rows) - 1, -1, -1)
        for i in order:
            cols, vals, dii = rows[i]
            x[i] = (b[i] - vals @ x[cols]) / dii

    def smooth(sm, k, b, x):                  # x None: zero guess
        As, d, _, _, bounds = mats[k]
        if sm.kind == _lib.SMOOTH_SGS:        # blas2.sgs_sweep at one leaf (blas2.py:113-162)
            x = np.zeros_like(b) if x is None else x
            halves = {0: (True, False), 1: (True,), 2: (False,)}[sm.direction]
            for _ in range(max(sm.sweeps, 1)):
                for fwd in halves:
                    gs_half(k, b, x, fwd)
            return x
        if sm.kind == _lib.SMOOTH_JACOBI:     # blas2.py:165-185
            if sm.weight == 0.0:
                return np.zeros_like(b) if x is None else x
            for _ in range(max(sm.sweeps, 1)):
                r = b if x is None else b - As @ x
                upd = sm.weight * (r / d[:, None])
                x = upd if x is None else x + upd
            return x
        lmin, lmax = bounds                   # solvers.py:520-571
        theta, delta = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
        sigma = theta / delta
        rho = 1.0 / sigma
        r = b if x is None else b - As @ x
        dv = r / (d[:, None] * theta)
        x = dv.copy() if x is None else x + dv
        for _ in range(max(sm.order, 1) - 1):
            r = r - As @ dv
            rho_new = 1.0 / (2.0 * sigma - rho)
            dv = dv * (rho_new * rho) + (2.0 * rho_new / delta) * (r / d[:, None])
            x = x + dv
            rho = rho_new
        return x

    def vcycle(k, b):
        if k == len(mats) - 1:
            return inv @ b
        As, d, P, R, _ = mats[k]
        x = smooth(pre, k, b, None)
        xc = vcycle(k + 1, R @ (b - As @ x))
        x = x + P @ xc
        return smooth(post, k, b, x)

    # columns in blocks: host memory stays O(n * block) however large n_l is
    n = mats[0][0].shape[0]
    T = np.empty((n, n))
    block = 512
    for j0 in range(0, n, block):
        j1 = min(n, j0 + block)
        E = np.zeros((n, j1 - j0))
        E[np.arange(j0, j1), np.arange(j1 - j0)] = 1.0
        T[:, j0:j1] = vcycle(0, E)
    return T
