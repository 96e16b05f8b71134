"""ctypes binding of libmrsolve_b200.so (the C ABI in include/mrsolve_b200.h).

The product path has no CPU fallback: if the library is missing it is built
(nvcc present) or the import fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import (BreakdownError, ConfigurationError, DeviceError, InstabilityError,
                     InvalidArgumentError, SetupDegeneracyError, SingularDiagonalError)

HERE = os.path.dirname(os.path.abspath(__file__))
# MRS_LIB: an alternative build of the same library (the checked variant,
# MRS_CHECKS=1 python -m paper_2103_07329_b200.build); default the in-tree one
LIBPATH = os.environ.get("MRS_LIB") or os.path.join(HERE, "libmrsolve_b200.so")

MRS_OK, MRS_ERR_ARG, MRS_ERR_CUDA, MRS_ERR_UNSUPPORTED, MRS_ERR_ALLOC = 0, 1, 2, 3, 4
MRS_ERR_BREAKDOWN, MRS_ERR_SINGULAR, MRS_ERR_DEGENERATE, MRS_ERR_STATE = 5, 6, 7, 8
MRS_ERR_INSTABILITY = 9

METHOD_CG, METHOD_BICGSTAB, METHOD_RBICGSTAB, METHOD_PBICGSTAB = 0, 1, 2, 3
METHOD_STATIONARY, METHOD_DIRECT = 4, 5
PC_NONE, PC_JACOBI, PC_MG, PC_SGS, PC_CHEB = 0, 1, 2, 3, 4
SMOOTH_JACOBI, SMOOTH_CHEBYSHEV, SMOOTH_SGS = 0, 1, 2
SGS_DIRECTIONS = {"symmetric": 0, "forward": 1, "backward": 2}


class mrs_csr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p),
                ("idx_bytes", C.c_int32), ("val_bytes", C.c_int32),
                ("slab_base", C.c_void_p), ("slab_shift", C.c_int32), ("pad_", C.c_int32),
                ("long_rows", C.c_void_p), ("n_long", C.c_int32), ("long_thr", C.c_int32),
                ("band", C.c_int32), ("blk_max", C.c_int32), ("flags", C.c_int32),
                ("pad2_", C.c_int32)]


class mrs_host_csr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p),
                ("idx_bytes", C.c_int32), ("val_bytes", C.c_int32),
                ("slab_base", C.c_void_p), ("slab_shift", C.c_int32), ("pad_", C.c_int32)]


class mrs_smoother(C.Structure):
    _fields_ = [("kind", C.c_int32), ("sweeps", C.c_int32), ("weight", C.c_double),
                ("order", C.c_int32), ("direction", C.c_int32)]


class mrs_plan_desc(C.Structure):
    _fields_ = [("method", C.c_int32), ("precond", C.c_int32), ("nrows", C.c_int64),
                ("m", C.c_int64), ("rel_tol", C.c_double), ("max_iters", C.c_int32),
                ("pc_weight", C.c_double), ("pc_sweeps", C.c_int32), ("mg_cycles", C.c_int32),
                ("pre", mrs_smoother), ("post", mrs_smoother), ("nlevels", C.c_int32),
                ("exec", C.c_int32), ("merged", C.c_int32), ("drift_limit", C.c_double),
                ("pc_direction", C.c_int32), ("vec32", C.c_int32)]


class mrs_stats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("status", C.c_int32),
                ("breakdown_column", C.c_int32), ("breakdown_site", C.c_int32),
                ("device_ms", C.c_double)]


class mrs_amg_params(C.Structure):
    _fields_ = [("strength_threshold", C.c_double), ("agg_num_levels", C.c_int32),
                ("num_paths", C.c_int32), ("coarse_matrix_size", C.c_int64),
                ("max_levels", C.c_int32), ("stall_ratio", C.c_double),
                ("mixed_precision", C.c_int32)]


_lib = None

#: symbol -> (restype, argtypes); every symbol include/mrsolve_b200.h declares
SIGNATURES = {
    "mrs_csr_spmv": (C.c_int, [C.POINTER(mrs_csr), C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                               C.c_void_p, C.c_void_p]),
    "mrs_csr_spmv_f32": (C.c_int, [C.POINTER(mrs_csr), C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                   C.c_void_p, C.c_void_p]),
    "mrs_axpby": (C.c_int, [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_void_p]),
    "mrs_add2_scaled": (C.c_int, [C.c_int64, C.c_int64] + [C.c_void_p] * 6),
    "mrs_fused_paired_update": (C.c_int, [C.c_int64, C.c_int64] + [C.c_void_p] * 9),
    "mrs_dot": (C.c_int, [C.c_int64, C.c_int64] + [C.c_void_p] * 4),
    "mrs_fused_update_dot": (C.c_int, [C.c_int64, C.c_int64] + [C.c_void_p] * 6),
    "mrs_fused_update_dot2": (C.c_int, [C.c_int64, C.c_int64] + [C.c_void_p] * 8),
    "mrs_gs_sweep": (C.c_int, [C.POINTER(mrs_csr), C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "mrs_plan_create": (C.c_int, [C.POINTER(mrs_plan_desc), C.POINTER(C.c_void_p)]),
    "mrs_plan_set_level": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(mrs_host_csr),
                                     C.POINTER(mrs_host_csr), C.POINTER(mrs_host_csr),
                                     C.c_double, C.c_double]),
    "mrs_plan_set_coarse_inverse": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "mrs_plan_set_dense_tail": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64]),
    "mrs_plan_finalize": (C.c_int, [C.c_void_p, C.c_void_p]),
    "mrs_plan_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                 C.c_void_p, C.POINTER(mrs_stats), C.c_void_p, C.c_void_p]),
    "mrs_plan_iteration_bytes": (C.c_double, [C.c_void_p]),
    "mrs_plan_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_int32,
                                   C.POINTER(C.c_int32)]),
    "mrs_plan_kernel_count": (C.c_int, [C.c_void_p]),
    "mrs_plan_launch_name": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_int32]),
    "mrs_plan_fixed_kernel_count": (C.c_int, [C.c_void_p]),
    "mrs_plan_destroy": (None, [C.c_void_p]),
    "mrs_amg_setup": (C.c_int, [C.POINTER(mrs_host_csr), C.POINTER(mrs_amg_params),
                                C.POINTER(C.c_void_p)]),
    "mrs_hier_nlevels": (C.c_int, [C.c_void_p]),
    "mrs_hier_get": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(mrs_host_csr)]),
    "mrs_hier_destroy": (None, [C.c_void_p]),
    "mrs_eig_bounds": (C.c_int, [C.POINTER(mrs_host_csr), C.c_int32, C.c_uint64, C.c_void_p,
                                 C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "mrs_status_string": (C.c_char_p, [C.c_int32]),
    "mrs_version": (C.c_int, []),
    "mrs_stream_launches": (C.c_int64, []),
    "mrs_galerkin_gpu_count": (C.c_int64, []),
    "mrs_set_option": (C.c_int, [C.c_char_p, C.c_int64]),
    "mrs_comm_unique_id": (C.c_int, [C.c_void_p]),
    "mrs_comm_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "mrs_comm_destroy": (None, [C.c_void_p]),
    "mrs_comm_create_loopback": (C.c_int, [C.c_int32, C.c_void_p]),
    "mrs_plan_set_comm": (C.c_int, [C.c_void_p, C.c_void_p]),
    "mrs_plan_set_layout": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int64]),
    "mrs_plan_set_halo": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_void_p,
                                    C.c_void_p, C.c_void_p]),
    "mrs_plan_set_interior": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int64]),
}


def lib():
    """Load the library, building it first when it is missing or stale."""
    global _lib
    if _lib is None:
        # torch first: its CUDA libraries bring their own libnccl.so.2, which
        # then also serves this library (same soname).  Loading ours first
        # would bind the system NCCL and break torch's newer NCCL symbols.
        import torch  # noqa: F401
        from . import build as _build
        if _build.needs_build():
            _build.build()
        if not os.path.exists(LIBPATH):
            raise ImportError(f"{LIBPATH} missing: the CUDA extension is required "
                              "(no CPU fallback)")
        L = C.CDLL(LIBPATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def set_option(key: str, value: int):
    """Tuning knob (see mrs_set_option in include/mrsolve_b200.h)."""
    check(lib().mrs_set_option(key.encode(), int(value)), f"set_option({key})")


def status_string(code: int) -> str:
    return lib().mrs_status_string(code).decode()


def check(code: int, what: str = "mrsolve_b200 call"):
    """Map a C status to the reference's exception types."""
    if code == MRS_OK:
        return
    msg = f"{what}: {status_string(code)}"
    if code == MRS_ERR_ARG:
        raise InvalidArgumentError(msg)
    if code == MRS_ERR_UNSUPPORTED:
        raise ConfigurationError(msg)
    if code == MRS_ERR_SINGULAR:
        raise SingularDiagonalError(msg)
    if code == MRS_ERR_DEGENERATE:
        raise SetupDegeneracyError(msg)
    if code == MRS_ERR_BREAKDOWN:
        raise BreakdownError(msg, -1)
    if code == MRS_ERR_INSTABILITY:
        raise InstabilityError(msg)
    raise DeviceError(msg, code)


#: index compression of plan uploads on the device (False / MRS_SLAB_ON_DEVICE=0:
#: core.slab_compress on the host, the round-1 path; identical result)
SLAB_ON_DEVICE = os.environ.get("MRS_SLAB_ON_DEVICE", "1") != "0"


def host_csr(blk, keep: list, slab=False) -> mrs_host_csr:
    """mrs_host_csr view of a CsrBlock-like object (arrays kept alive in `keep`).
    ``slab=True``: store 32-bit column indices as slab-relative 16-bit ones
    when every slab's column span fits (core.slab_compress)."""
    import numpy as np
    rp = np.ascontiguousarray(blk.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(blk.col_idx)
    if ci.dtype not in (np.uint8, np.uint16, np.uint32):
        ci = ci.astype(np.uint32)
    v = np.ascontiguousarray(blk.values)
    if v.dtype not in (np.float32, np.float64):
        v = v.astype(np.float64)
    base_p, shift = None, 0
    flags = 0
    if slab and ci.dtype == np.uint32:
        if SLAB_ON_DEVICE:
            flags = 1           # the upload compresses on the GPU (csrc/slab.cu, same rule)
        else:
            from .core import slab_compress
            sc = slab_compress(rp, ci)
            if sc is not None:
                ci, base, shift = sc
                keep.append(base)
                base_p = base.ctypes.data
    keep.extend([rp, ci, v])
    return mrs_host_csr(int(blk.nrows), int(blk.ncols), int(rp[-1]), rp.ctypes.data,
                        ci.ctypes.data, v.ctypes.data, ci.dtype.itemsize, v.dtype.itemsize,
                        base_p, shift, flags)
