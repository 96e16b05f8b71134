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
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import CsrBlock, PrecisionTag, as_csr, choose_width
from .errors import InvalidArgumentError, SingularDiagonalError

__all__ = ["AmgParams", "Level", "Hierarchy", "setup", "estimate_eig_bounds", "coarse_inverse"]


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
