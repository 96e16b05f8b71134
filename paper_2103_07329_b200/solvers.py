"""Solver composition on the GPU: ``prepare(config, A).run(B, X) -> SolveStats``.

Drop-in for the reference's solve path (/root/reference/pkg/src/mrsolve/
solvers.py:850-959): same ParamTree configuration, same SolveStats fields,
same exception types.  ``prepare`` does all setup -- validation, the AMG
hierarchy (native restatement of amg.setup, or a hierarchy passed in),
Chebyshev eigenvalue bounds, the dense coarse inverse -- and uploads it
once; ``run`` executes one whole solve on the device as a single CUDA graph
launch (iteration loop driven on the device; see csrc/solver.cu).

Device path: solver CG or BiCGStab in its
three formulations -- classical, reordered (RBiCGStab), pipelined
(PBiCGStab); merged=0/1 --, MultiGrid as a solver, the stationary Jacobi /
Gauss-Seidel solvers and Direct (dense inverse); preconditioner none /
Jacobi / Gauss-Seidel / Chebyshev / MultiGrid V-cycle; smoothers Jacobi,
Chebyshev or (hybrid, one-leaf) Gauss-Seidel -- the reference's default
MultiGrid smoother, run in its exact sequential order by level scheduling.
The one composition the reference's ParamTree can express that is not on the
device path -- a Krylov method (BiCGStab) as preconditioner or smoother --
raises ConfigurationError; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .amg import (AmgParams, Hierarchy, coarse_inverse, dense_tail_level, estimate_eig_bounds,
                  setup as amg_setup, vcycle_tail_operator)
from .core import BlockVector, PrecisionTag, as_csr
from .errors import (BreakdownError, ConfigurationError, InvalidArgumentError,
                     ShapeMismatchError)
from .params import METHOD_FAMILIES, ParamTree

__all__ = ["SolveStats", "ConfiguredSolver", "prepare", "solve", "DevicePlan", "DRIFT_LIMIT"]

#: pipelined BiCGStab drift limit (solvers.py:68): ||r_init - op(zacc)|| over
#: the recurrence norm above this raises InstabilityError.  Read at prepare().
DRIFT_LIMIT = 1e3

_BREAK_MSG = {
    1: "CG search-direction curvature vanished",
    2: "CG rho vanished",
    3: "BiCGStab (r0, Ap) vanished",
    4: "BiCGStab stabilization step vanished",
    5: "BiCGStab rho vanished",
    6: "BiCGStab omega vanished",
    7: "BiCGStab (r0, Ar) vanished",
    8: "BiCGStab (r0, s) vanished",
}


@dataclass
class SolveStats:
    """solvers.py:80-92."""

    iterations: int
    converged: np.ndarray
    final_rel_residual: np.ndarray
    residual_history: list = field(default_factory=list)
    method: str = ""
    device_ms: float = 0.0

    @property
    def all_converged(self) -> bool:
        return bool(np.all(self.converged))


@dataclass
class ConfiguredSolver:
    method: str
    run: object
    hierarchy: Hierarchy | None = None
    plan_factory: object = None
    desc: object = None          # plan descriptor (without m)
    levels: list | None = None   # [(A, P, R)] as uploaded

    def minimal_iteration_bytes(self, m: int) -> float:
        """SURVEY.md 8(d) minimal bytes of one outer iteration (byte_model);
        the plan's own model (incl. the collapsed dense tail) is
        ``plan_factory(m).iteration_bytes``."""
        from .byte_model import iteration_bytes_minimal
        return iteration_bytes_minimal(self.desc, self.levels, m)


def _sgs_direction(plist) -> int:
    d = plist.get_str("direction")
    if d not in _lib.SGS_DIRECTIONS:          # blas2.py:125-126
        raise InvalidArgumentError(f"unknown sweep direction {d!r}")
    return _lib.SGS_DIRECTIONS[d]


def _smoother(plist) -> _lib.mrs_smoother:
    if plist is None:
        # the reference's MultiGrid default: one symmetric hybrid Gauss-Seidel
        # sweep (solvers.py:609-612, :630-631)
        return _lib.mrs_smoother(_lib.SMOOTH_SGS, 1, 0.0, 0, _lib.SGS_DIRECTIONS["symmetric"])
    if plist.method == "Jacobi":
        return _lib.mrs_smoother(_lib.SMOOTH_JACOBI, plist.get_int("max_iters"),
                                 plist.get_float("weight"), 0, 0)
    if plist.method == "Chebyshev":
        order = plist.get_int("polynomial_order")
        if order < 1:
            raise InvalidArgumentError("polynomial_order must be >= 1")
        return _lib.mrs_smoother(_lib.SMOOTH_CHEBYSHEV, 1, 0.0, order, 0)
    if plist.method == "Gauss-Seidel":
        return _lib.mrs_smoother(_lib.SMOOTH_SGS, plist.get_int("max_iters"), 0.0, 0,
                                 _sgs_direction(plist))
    raise ConfigurationError(f"smoother {plist.method!r} is not on the device path")


class CoarseOps:
    """Dense operators of the coarse end of the V-cycle (uploaded once):
    ``inv`` = inverse of the coarsest operator, ``tail`` = the collapsed
    sub-V-cycle operator of level ``tail_level`` (amg.vcycle_tail_operator),
    or None."""

    def __init__(self, inv, tail_level=-1, tail=None):
        self.inv, self.tail_level, self.tail = inv, tail_level, tail


class DevicePlan:
    """One uploaded solver instance for a fixed RHS count m (owns a C plan)."""

    #: store 32-bit level indices as slab-relative 16-bit ones where they fit
    compress_indices = True

    def __init__(self, desc: _lib.mrs_plan_desc, levels, inv, method_name: str, dist=None):
        self.L = _lib.lib()
        self.desc = desc
        self.method = method_name
        h = C.c_void_p()
        _lib.check(self.L.mrs_plan_create(C.byref(desc), C.byref(h)), "plan create")
        self.h = h
        try:
            if dist is not None:
                team, lays = dist
                _lib.check(self.L.mrs_plan_set_comm(h, team.comm), "plan set_comm")
                for l, lay in enumerate(lays):
                    _lib.check(self.L.mrs_plan_set_layout(h, l, int(lay.replicated),
                                                          int(lay.slice[0]), int(lay.slice[1])),
                               f"layout level {l}")
                    for which, hp in lay.halos.items():
                        _lib.check(self.L.mrs_plan_set_halo(
                            h, l, which, hp.nsend, hp.send_idx.ctypes.data,
                            hp.send_counts.ctypes.data, hp.recv_counts.ctypes.data),
                            f"halo level {l}/{which}")
                    for which, (ilo, ihi) in getattr(lay, "interior", {}).items():
                        _lib.check(self.L.mrs_plan_set_interior(h, l, which, ilo, ihi),
                                   f"interior rows level {l}/{which}")
            for l, (A, P, R, bounds) in enumerate(levels):
                keep: list = []
                sl = DevicePlan.compress_indices
                a = _lib.host_csr(A, keep, sl)
                p = _lib.host_csr(P, keep, sl) if P is not None else None
                r = _lib.host_csr(R, keep, sl) if R is not None else None
                lo, hi = bounds if bounds is not None else (0.0, 0.0)
                _lib.check(self.L.mrs_plan_set_level(h, l, C.byref(a),
                                                     C.byref(p) if p is not None else None,
                                                     C.byref(r) if r is not None else None,
                                                     float(lo), float(hi)), f"upload level {l}")
            tail = None
            if isinstance(inv, CoarseOps):
                inv, tail = inv.inv, inv
            if inv is not None:
                inv = np.ascontiguousarray(inv, dtype=np.float64)
                _lib.check(self.L.mrs_plan_set_coarse_inverse(h, inv.ctypes.data, inv.shape[0]),
                           "coarse inverse")
            if tail is not None and tail.tail is not None and (
                    dist is None or dist[1][tail.tail_level].replicated):
                T = np.ascontiguousarray(tail.tail, dtype=np.float64)
                _lib.check(self.L.mrs_plan_set_dense_tail(h, tail.tail_level, T.ctypes.data,
                                                          T.shape[0]), "dense V-cycle tail")
            _lib.check(self.L.mrs_plan_finalize(h, None), "plan finalize")
        except Exception:
            self.L.mrs_plan_destroy(h)
            self.h = None
            raise

    def __del__(self):
        if getattr(self, "h", None):
            try:
                self.L.mrs_plan_destroy(self.h)
            except Exception:
                pass
            self.h = None

    @property
    def iteration_bytes(self) -> float:
        return self.L.mrs_plan_iteration_bytes(self.h)

    @property
    def kernels_per_iteration(self) -> int:
        return self.L.mrs_plan_kernel_count(self.h)

    def profile(self, iters: int = 3, B=None) -> np.ndarray:
        """Warm per-launch times (us) of one iteration body (diagnostics).
        ``B``: CUDA tensor of right-hand sides (None: the plan's staging copy,
        i.e. the last solve run from host buffers)."""
        import torch
        out = np.zeros(512)
        n = C.c_int32()
        bp = C.c_void_p(B.data_ptr()) if B is not None else None
        _lib.check(self.L.mrs_plan_profile(self.h, bp, iters,
                                           C.c_void_p(torch.cuda.current_stream().cuda_stream),
                                           out.ctypes.data, 512, C.byref(n)), "profile")
        return out[:n.value].copy()

    def launch_names(self) -> list:
        """Demangled kernel name of every iteration-body launch (diagnostics)."""
        import subprocess
        out = []
        buf = C.create_string_buffer(512)
        for i in range(self.kernels_per_iteration):
            _lib.check(self.L.mrs_plan_launch_name(self.h, i, buf, 512), "launch name")
            out.append(buf.value.decode())
        try:
            dem = subprocess.run(["c++filt"], input="\n".join(out), capture_output=True,
                                 text=True, timeout=10).stdout.splitlines()
            if len(dem) == len(out):
                out = dem
        except Exception:
            pass
        return out

    def kernel_launches(self, iterations: int) -> int:
        """Kernels one solve of `iterations` iterations launches."""
        return self.L.mrs_plan_fixed_kernel_count(self.h) + iterations * self.kernels_per_iteration

    def solve(self, Bp: int, Xp: int, x_zero: bool, host: bool, stream=None):
        m, maxit = int(self.desc.m), int(self.desc.max_iters)
        st = _lib.mrs_stats()
        rel = np.zeros(m)
        hist = np.zeros((maxit + 1) * m)
        rc = self.L.mrs_plan_solve(self.h, Bp, Xp, int(bool(x_zero)), int(bool(host)), stream,
                                   C.byref(st), rel.ctypes.data, hist.ctypes.data)
        if rc == _lib.MRS_ERR_BREAKDOWN:
            raise BreakdownError(_BREAK_MSG.get(st.breakdown_site, "Krylov breakdown"),
                                 column=int(st.breakdown_column))
        _lib.check(rc, "solve")
        it = int(st.iterations)
        history = [hist[i * m:(i + 1) * m].copy() for i in range(it + 1)]
        tol = float(self.desc.rel_tol)
        if int(self.desc.method) == _lib.METHOD_DIRECT:   # solvers.py:598-604
            return SolveStats(1, rel <= 1e-8, rel, [rel.copy()], self.method, float(st.device_ms))
        return SolveStats(it, rel <= tol, rel, history, self.method, float(st.device_ms))


def _vector_args(B, X):
    """Resolve (B, X) into pointers: host BlockVectors/ndarrays or CUDA tensors."""
    try:
        import torch
        is_t = isinstance(B, torch.Tensor)
    except ImportError:       # pragma: no cover
        is_t = False
    if is_t:
        import torch
        for t, nm in ((B, "B"), (X, "X")):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                    and t.dim() == 2 and t.is_contiguous()):
                raise InvalidArgumentError(f"{nm} must be a contiguous (n, m) float64 CUDA tensor")
        if B.shape != X.shape:
            raise ShapeMismatchError(f"block vector shapes differ: {tuple(B.shape)} vs {tuple(X.shape)}")
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        return B.shape, B.data_ptr(), X.data_ptr(), False, False, stream, None
    Bv = B if hasattr(B, "flags") and hasattr(B, "data") else BlockVector.from_array(B)
    if not (hasattr(X, "flags") and hasattr(X, "data")):
        raise InvalidArgumentError("X must be a BlockVector (or CUDA tensor)")
    if Bv.data.shape != X.data.shape:
        raise ShapeMismatchError(f"block vector shapes differ: {Bv.data.shape} vs {X.data.shape}")
    if not Bv.flags.initialized:
        raise InvalidArgumentError("residual needs an initialized right-hand side")
    b = np.ascontiguousarray(Bv.data, dtype=np.float64)
    if not X.data.flags.c_contiguous or X.data.dtype != np.float64:
        raise InvalidArgumentError("X data must be C-contiguous float64")
    x_zero = bool(X.flags.zero)
    if not x_zero and not X.flags.initialized:
        raise InvalidArgumentError("residual input vector is not initialized")
    import torch
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return b.shape, b.ctypes.data, X.data.ctypes.data, x_zero, True, stream, (b, X)


def prepare(config: ParamTree, A, team=None, *, hierarchy=None, exec_mode: str = "graph",
            eig_bounds=None) -> ConfiguredSolver:
    """Build the device solver combination described by ``config``.

    ``hierarchy``: optional pre-built hierarchy (ours or a reference
    ``amg.Hierarchy``); otherwise the native reference setup runs here.
    ``exec_mode``: "graph" (default, device-driven loop) or "eager".
    ``team``: a :class:`~paper_2103_07329_b200.team.GpuTeam` for the
    row-partitioned multi-GPU path (None = this process's current GPU).
    """
    if team is not None and hasattr(team, "agg_rows_per_rank"):   # GpuTeam (a reference
        from .team import prepare_distributed                      # WorkerTeam is ignored)
        return prepare_distributed(config, A, team, hierarchy=hierarchy, exec_mode=exec_mode,
                                   eig_bounds=eig_bounds)
    desc, levels, inv, h, name, Ab = _configure(config, A, hierarchy, exec_mode, eig_bounds)
    return _prepare_single(desc, levels, inv, h, name, Ab, config.role("solver").method)


def _configure(config, A, hierarchy, exec_mode, eig_bounds):
    """Validate the configuration and build everything that is uploaded:
    plan descriptor, per-level (A, P, R, Chebyshev bounds), coarse inverse,
    hierarchy, method name (solvers.py:864-953)."""
    if not config.finalized:
        config.set_defaults()
    violations = config.validate()
    if violations:
        raise ConfigurationError("; ".join(violations))
    Ab = as_csr(A)
    if Ab.nrows != Ab.ncols:
        raise InvalidArgumentError("the system matrix must be square")
    sp = config.role("solver")
    method = sp.method
    family = METHOD_FAMILIES[method]
    if family not in ("CG", "BiCGStab", "MultiGrid", "Jacobi", "Gauss-Seidel", "Direct"):
        raise ConfigurationError(f"method {method!r} cannot act as a solver")   # solvers.py:953
    if family == "Direct":            # no iteration keys (direct_solve tests rel <= 1e-8)
        tol, iters = 1e-8, 0
    else:
        tol = sp.get_float("rel_tolerance")
        iters = sp.get_int("max_iters")
    merged = bool(sp.get_int("merged")) if family == "BiCGStab" else False
    # SolveStats.method as the reference names it (solvers.py:292, :363, :478;
    # the stationary and direct families report the configured method)
    name = ("CG" if family == "CG" else
            method + ("/merged" if merged else "") if family == "BiCGStab" else method)

    pl = config.role("preconditioner")
    if family == "MultiGrid":
        if pl is not None:                       # solvers.py:904-905
            raise ConfigurationError("MultiGrid solver takes no preconditioner")
        pl = sp                                  # the solver role carries the mg_* keys
    elif family in ("Jacobi", "Gauss-Seidel", "Direct"):
        pl = None                                # built but unused by the reference
    desc = _lib.mrs_plan_desc()
    desc.method = {"CG": _lib.METHOD_CG, "BiCGStab": _lib.METHOD_BICGSTAB,
                   "RBiCGStab": _lib.METHOD_RBICGSTAB, "PBiCGStab": _lib.METHOD_PBICGSTAB,
                   "MultiGrid": _lib.METHOD_STATIONARY, "Jacobi": _lib.METHOD_STATIONARY,
                   "Gauss-Seidel": _lib.METHOD_STATIONARY,
                   "Direct": _lib.METHOD_DIRECT}[method if family == "BiCGStab" else family]
    desc.drift_limit = DRIFT_LIMIT
    desc.nrows = Ab.nrows
    desc.rel_tol = tol
    desc.max_iters = iters
    desc.exec = 0 if exec_mode == "graph" else 1
    desc.merged = int(merged)
    desc.mg_cycles = 1
    desc.nlevels = 1
    levels, inv, h = None, None, None
    if family == "Direct":                       # direct_solve (solvers.py:588-604)
        desc.precond = _lib.PC_NONE
        desc.max_iters = 0
        levels = [(Ab, None, None, None)]
        inv = coarse_inverse(Ab)
    elif family == "Jacobi":                     # _stationary_solve with one sweep per step
        desc.precond = _lib.PC_JACOBI
        desc.pc_weight = sp.get_float("weight")
        desc.pc_sweeps = 1
        levels = [(Ab, None, None, None)]
    elif family == "Gauss-Seidel":
        desc.precond = _lib.PC_SGS
        desc.pc_sweeps = 1
        desc.pc_direction = _sgs_direction(sp)
        levels = [(Ab, None, None, None)]
    elif pl is None:
        desc.precond = _lib.PC_NONE
        levels = [(Ab, None, None, None)]
    elif pl.method == "Chebyshev":               # _SweepPrecond(chebyshev_apply), :796-802
        desc.precond = _lib.PC_CHEB
        order = pl.get_int("polynomial_order")
        if order < 1:
            raise InvalidArgumentError("polynomial_order must be >= 1")
        desc.pre = _lib.mrs_smoother(_lib.SMOOTH_CHEBYSHEV, 1, 0.0, order, 0)
        bounds = tuple(eig_bounds[0]) if eig_bounds is not None else estimate_eig_bounds(Ab)
        if not (0.0 < bounds[0] < bounds[1]):
            raise InvalidArgumentError(
                f"eigenvalue bounds must satisfy 0 < lmin < lmax, got {bounds}")
        levels = [(Ab, None, None, bounds)]
    elif pl.method == "Jacobi":
        desc.precond = _lib.PC_JACOBI
        desc.pc_weight = pl.get_float("weight")
        desc.pc_sweeps = pl.get_int("max_iters")
        levels = [(Ab, None, None, None)]
    elif pl.method == "Gauss-Seidel":            # _SweepPrecond(sgs_sweep), solvers.py:792-797
        desc.precond = _lib.PC_SGS
        desc.pc_sweeps = pl.get_int("max_iters")
        desc.pc_direction = _sgs_direction(pl)
        levels = [(Ab, None, None, None)]
    elif pl.method == "MultiGrid":
        if pl.get_str("mg_cycle") != "V":
            raise ConfigurationError("only the V cycle is implemented")
        desc.precond = _lib.PC_MG
        # preconditioner: max_iters V-cycles per application; solver: one per step
        desc.mg_cycles = 1 if family == "MultiGrid" else max(pl.get_int("max_iters"), 1)
        desc.pre = _smoother(config.role("pre_smoother"))
        desc.post = _smoother(config.role("post_smoother"))
        # extension (not in the reference schema): fp32 V-cycle vectors below
        # level 0 -- the north star's "fp32 preconditioner" (csrc/solver.cu vec32)
        try:
            vprec = pl.get_str("mg_vector_precision")
        except Exception:            # a reference ParamTree has no such key
            vprec = "fp64"
        if vprec not in ("fp64", "fp32", "fp32_all"):
            raise InvalidArgumentError(
                f"mg_vector_precision must be fp64, fp32 or fp32_all, got {vprec!r}")
        # fp32: V-cycle vectors below level 0; fp32_all: level 0's too (the whole
        # preconditioner on float vectors, Krylov vectors fp64)
        desc.vec32 = {"fp64": 0, "fp32": 1, "fp32_all": 2}[vprec]
        if hierarchy is None:
            params = AmgParams(strength_threshold=pl.get_float("mg_strength_threshold"),
                               agg_num_levels=pl.get_int("mg_agg_num_levels"),
                               num_paths=pl.get_int("mg_num_paths"),
                               coarse_matrix_size=pl.get_int("mg_coarse_matrix_size"),
                               max_levels=pl.get_int("mg_max_levels"))
            h = amg_setup(Ab, params, mixed_precision=bool(pl.get_int("mg_mixed_precision")))
        else:
            h = Hierarchy.of(hierarchy)
        cheb = _lib.SMOOTH_CHEBYSHEV in (desc.pre.kind, desc.post.kind)
        levels = []
        for l, lv in enumerate(h.levels):
            bounds = None
            if cheb and l < h.nlevels - 1:
                if eig_bounds is not None:
                    lv.eig_bounds = tuple(eig_bounds[l])
                if lv.eig_bounds is None:
                    lv.eig_bounds = estimate_eig_bounds(lv.A)
                bounds = lv.eig_bounds
                lmin, lmax = bounds
                if not (0.0 < lmin < lmax):
                    raise InvalidArgumentError(
                        f"eigenvalue bounds must satisfy 0 < lmin < lmax, got {bounds}")
            levels.append((lv.A, lv.P, lv.R, bounds))
        inv = coarse_inverse(h.coarsest.A)
        h.coarsest.lu = inv
        desc.nlevels = h.nlevels
        tl = dense_tail_level(levels, pre=desc.pre, post=desc.post)
        if tl >= 0:
            T = tail_operator(levels, tl, desc.pre, desc.post, inv)
            if T is not None:
                inv = CoarseOps(inv, tl, T)
    else:
        raise ConfigurationError(f"preconditioner {pl.method!r} is not on the device path")
    return desc, levels, inv, h, name, Ab


#: where the collapsed tail's dense operator is built: "device" (default when a
#: GPU is present) or "host" (amg.vcycle_tail_operator: scipy products; the CPU
#: tests and MRS_TAIL_BUILD=host)
TAIL_BUILD = os.environ.get("MRS_TAIL_BUILD", "device")


def tail_operator(levels, start, pre, post, inv):
    """Dense operator of the sub-V-cycle below level ``start`` (setup phase)."""
    if TAIL_BUILD == "device":
        try:
            import torch
            on_gpu = torch.cuda.is_available()
        except Exception:
            on_gpu = False
        if on_gpu:
            return tail_operator_device(levels, start, pre, post, inv)
    return vcycle_tail_operator(levels, start, pre, post, inv)


def tail_operator_device(levels, start: int, pre, post, inv, cols: int = 64):
    """amg.vcycle_tail_operator on the GPU: the sub-hierarchy from level
    ``start`` is uploaded as a MultiGrid-as-solver plan and ONE V-cycle from a
    zero guess is applied to the n_l unit vectors, ``cols`` right-hand sides
    at a time, with the plan's own per-level kernels (SpMM, fused smoothers,
    level-scheduled Gauss-Seidel, dense coarse solve) -- the exact kernels the
    collapsed tail replaces in the solve.  Replaces minutes of scipy products
    on the host for the tail levels of large hierarchies (the dominant part of
    ``prepare`` at C4 sizes).  Returns the (n_l, n_l) float64 array."""
    import torch
    for sm in (pre, post):
        if sm.kind not in (_lib.SMOOTH_JACOBI, _lib.SMOOTH_CHEBYSHEV, _lib.SMOOTH_SGS):
            return None
    sub = list(levels[start:])
    n = as_csr(sub[0][0]).nrows
    d = _lib.mrs_plan_desc()
    d.method = _lib.METHOD_STATIONARY
    d.precond = _lib.PC_MG
    d.nrows = n
    d.m = cols
    d.rel_tol = 0.0                      # never "converged": exactly max_iters = 1 cycle
    d.max_iters = 1
    d.exec = 1
    d.mg_cycles = 1
    d.pre, d.post = pre, post
    d.nlevels = len(sub)
    d.drift_limit = DRIFT_LIMIT
    plan = DevicePlan(d, sub, inv, "tail-builder")
    try:
        dev = torch.device("cuda", torch.cuda.current_device())
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        T = torch.empty((n, n), dtype=torch.float64, device=dev)
        B = torch.empty((n, cols), dtype=torch.float64, device=dev)
        X = torch.empty((n, cols), dtype=torch.float64, device=dev)
        lanes = torch.arange(cols, device=dev)
        for j0 in range(0, n, cols):
            w = min(cols, n - j0)
            # unit vectors e_j0 .. e_j0+w-1 (the last block repeats its last column)
            B.zero_()
            B[torch.clamp(lanes + j0, max=n - 1), lanes] = 1.0
            X.zero_()
            plan.solve(B.data_ptr(), X.data_ptr(), True, False, stream)
            T[:, j0:j0 + w] = X[:, :w]
        out = T.cpu().numpy()
    finally:
        del plan
    return out


def _prepare_single(desc, levels, inv, h, name, Ab, method):
    plans: dict = {}

    def plan_for(m: int) -> DevicePlan:
        if m not in plans:
            d = _lib.mrs_plan_desc.from_buffer_copy(desc)
            d.m = m
            plans[m] = DevicePlan(d, levels, inv, name)
        return plans[m]

    def run(B, X, x_is_zero=None) -> SolveStats:
        """Solve in place on X.  Host BlockVectors: the zero flag of X selects the
        zero-guess path (like the reference); CUDA tensors: pass x_is_zero."""
        shape, bp, xp, x_zero, host, stream, keep = _vector_args(B, X)
        if x_is_zero is not None:
            x_zero = bool(x_is_zero)
        if shape[0] != Ab.nrows:
            raise ShapeMismatchError(f"vector has {shape[0]} rows, matrix has {Ab.nrows}")
        if shape[1] > 64:
            raise InvalidArgumentError("at most 64 right-hand sides per solve")
        stats = plan_for(shape[1]).solve(bp, xp, x_zero, host, stream)
        if host:
            X.flags.zero = False
            X.flags.initialized = True
        return stats

    return ConfiguredSolver(method, run, h, plan_for, desc,
                            [(lv[0], lv[1], lv[2]) for lv in levels])


def solve(config: ParamTree, A, B, X, team=None) -> SolveStats:
    """Prepare and run (solvers.py:956-959)."""
    return prepare(config, A, team).run(B, X)
