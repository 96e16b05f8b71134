"""SURVEY.md 8(d) minimal byte model of one outer solver iteration.

The roofline denominator of a whole solve: the bytes an ideal implementation
of the reference's algorithm must move per iteration -- every SpMM streams its
matrix once (sizes as uploaded: int32 row pointers, 16/32-bit or slab-relative
16-bit columns, f64/f32 values) and reads/writes its vectors once, plus the
minimal vector passes of the Krylov method (SURVEY.md 8(d) "Algorithmic
bytes: solver").  It is deliberately independent of this implementation's
choices: the collapsed dense V-cycle tail (n_l^2 * 8 bytes streamed per
application instead of the sparse coarse levels it replaces), fused seeds and
dots are NOT counted here -- that is the plan's own model
(``DevicePlan.iteration_bytes``, csrc/solver.cu).

    V = n * m * s_vec  (s_vec = 8; 4 on fp32-vector levels)
    PCG + preconditioner M:   mat(A0) + 13 V           + bytes(M)
    Jacobi-PCG (M = 1 sweep): mat(A0) + 11 V + 16 n    (z = r / d recomputed)
    BiCGStab:               2 mat(A0) + 21 V           + 2 bytes(M)
    V(1,1) per level l < L-1 (V = V_l, Vc = V_{l+1}):
      Jacobi pre  2V + 8n (zero guess: x = w b / d) ... then residual mat(A)+3V
      restrict mat(R) + V + Vc, prolong mat(P) + Vc + 2V, post mat(A) + 3V + 8n
      Chebyshev-2 pre mat(A) + 5V + 16n, post 2 mat(A) + 9V + 16n
    coarsest: n_c^2 * 8 + 2 Vc
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import as_csr, slab_compress

__all__ = ["mat_bytes", "iteration_bytes_minimal"]


def mat_bytes(M, slab: bool = True) -> float:
    """Bytes of one pass over a CSR block as the device stores it."""
    M = as_csr(M)
    n, nnz = M.nrows, M.nnz
    vb = M.values.dtype.itemsize
    ib = max(2, M.col_idx.dtype.itemsize)        # u8 is widened to u16 at upload
    extra = 0
    if slab and M.col_idx.dtype.itemsize == 4 and nnz:
        sc = slab_compress(M.row_ptr, M.col_idx)
        if sc is not None:
            ib = 2
            extra = sc[1].nbytes
    return float(nnz * (vb + ib) + (n + 1) * 4 + extra)


def _smoother_bytes(sm, A, n, V, pre: bool) -> float:
    matA = mat_bytes(A)
    if sm.kind == _lib.SMOOTH_CHEBYSHEV:
        # step 1: zero guess x = dv = b/(d theta): read b, write x (2V); nonzero
        # x: r = b - A x, x += dv, and r, dv kept for step 2 when there is one.
        # step j >= 2: gather dv, read r, read x (not at j = 2 after a zero
        # guess: x is dv), write x, and r, dv again unless it is the last step.
        k = max(int(sm.order), 1)
        total = (2 * V + 8 * n) if pre else (matA + 3 * V + (2 * V if k > 1 else 0) + 8 * n)
        for j in range(2, k + 1):
            total += matA + 3 * V + (0 if (pre and j == 2) else V) + \
                (2 * V if j < k else 0) + 8 * n
        return total
    if sm.kind == _lib.SMOOTH_JACOBI:
        s = max(int(sm.sweeps), 1)
        if sm.weight == 0.0:
            return 0.0
        first = (2 * V + 8 * n) if pre else (matA + 3 * V + 8 * n)
        return first + (s - 1) * (matA + 3 * V + 8 * n)
    # Gauss-Seidel: one matrix pass + b, x read, x written per half-sweep
    halves = 2 if sm.direction == 0 else 1
    return max(int(sm.sweeps), 1) * halves * (matA + 3 * V + 8 * n)


def _vcycle_bytes(levels, m, pre, post, vec32_end=0) -> float:
    """One V(1,1) cycle from level 0 with a zero initial guess."""
    total = 0.0
    L = len(levels)
    for l, (A, P, R) in enumerate(levels):
        s = 4 if 1 <= l < vec32_end else 8
        n = as_csr(A).nrows
        V = n * m * s
        if l == L - 1:
            total += n * n * 8.0 + 2 * V
            break
        nc = as_csr(levels[l + 1][0]).nrows
        sc = 4 if 1 <= l + 1 < vec32_end else 8
        Vc = nc * m * sc
        total += _smoother_bytes(pre, A, n, V, pre=True)
        total += mat_bytes(A) + 3 * V                      # residual r = b - A x
        total += mat_bytes(R) + V + Vc                     # restriction
        total += mat_bytes(P) + Vc + 2 * V                 # prolongation x += P xc
        total += _smoother_bytes(post, A, n, V, pre=False)
    return total


def iteration_bytes_minimal(desc, levels, m: int) -> float:
    """Minimal bytes of one outer iteration.  ``desc``: the plan descriptor
    (_lib.mrs_plan_desc); ``levels``: [(A, P, R)] as uploaded (level 0 only
    for single-level preconditioners)."""
    A0 = levels[0][0]
    n = as_csr(A0).nrows
    V = n * m * 8.0
    matA = mat_bytes(A0)
    if desc.precond == _lib.PC_MG:
        end = len(levels) - 1 if getattr(desc, "vec32", 0) else 0
        pc = _vcycle_bytes(levels, m, desc.pre, desc.post, end) * max(int(desc.mg_cycles), 1)
    elif desc.precond == _lib.PC_JACOBI:
        pc = _smoother_bytes(_lib.mrs_smoother(_lib.SMOOTH_JACOBI, desc.pc_sweeps,
                                               desc.pc_weight, 0, 0), A0, n, V, pre=True)
    elif desc.precond == _lib.PC_CHEB:
        pc = _smoother_bytes(desc.pre, A0, n, V, pre=True)
    elif desc.precond == _lib.PC_SGS:
        pc = _smoother_bytes(_lib.mrs_smoother(_lib.SMOOTH_SGS, desc.pc_sweeps, 0.0, 0,
                                               desc.pc_direction), A0, n, V, pre=True)
    else:
        pc = 0.0
    if desc.method == _lib.METHOD_CG:
        if desc.precond == _lib.PC_JACOBI and desc.pc_sweeps <= 1:
            return matA + 11 * V + 16 * n                  # z = r / d recomputed
        return matA + 13 * V + pc
    if desc.method in (_lib.METHOD_BICGSTAB, _lib.METHOD_RBICGSTAB, _lib.METHOD_PBICGSTAB):
        return 2 * matA + 21 * V + 2 * pc
    # stationary: one preconditioner step + the true residual and its norm
    return pc + matA + 4 * V
