"""Device kernel plugin: the `mrsolve.kernels` module interface on CUDA tensors.

Same function names, argument meaning and arithmetic as the reference plugin
(/root/reference/pkg/src/mrsolve/kernels/__init__.py:27-41, compiled twin
kernels/_ckernels.pyx), executed by the sm_100a kernels of
libmrsolve_b200.so on torch's current CUDA stream:

* vectors: (n, m) float64 CUDA tensors, row-major (RHS-interleaved);
* matrix arrays: CUDA tensors -- row_ptr int32 (int64 accepted, converted),
  col_idx uint8/uint16/uint32 (int16/int32 bit patterns accepted), values
  float32/float64;
* per-column scalars: python floats, sequences or (m,) tensors;
* ``dot_partial`` and the fused dots return (m,) float64 CUDA tensors.

There is no CPU fallback: non-CUDA inputs raise ``InvalidArgumentError``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgumentError, ShapeMismatchError

__all__ = ["BACKEND", "MODE_ASSIGN", "MODE_ADD", "MODE_SUB", "MODE_RSUB", "DeviceCsr",
           "csr_spmv", "axpby", "add2_scaled", "dot_partial", "fused_update_dot",
           "fused_paired_update", "fused_update_dot2", "gs_sweep"]

BACKEND = "cuda-sm100a"
MODE_ASSIGN, MODE_ADD, MODE_SUB, MODE_RSUB = 0, 1, 2, 3

_IDX_BYTES = {torch.uint8: 1, torch.uint16: 2, torch.int16: 2, torch.uint32: 4, torch.int32: 4}
_VAL_BYTES = {torch.float32: 4, torch.float64: 8}


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _vec(t, name, dtype=torch.float64):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidArgumentError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype or t.dim() != 2 or not t.is_contiguous():
        raise InvalidArgumentError(f"{name} must be a contiguous (n, m) {dtype} tensor")
    return t


def _scal(a, m, dev):
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=torch.float64).reshape(-1)
    else:
        t = torch.as_tensor(np.asarray(a, dtype=np.float64).reshape(-1), device=dev)
    if t.numel() == 1:
        t = t.expand(m)
    if t.numel() != m:
        raise InvalidArgumentError(f"expected {m} per-RHS scalars, got {t.numel()}")
    return t.contiguous()


def _ck(code, what):
    _lib.check(code, what)


class DeviceCsr:
    """A CSR block resident on the GPU (int32 row pointers)."""

    def __init__(self, row_ptr, col_idx, values, nrows, ncols, device=None, slab=False):
        """``slab=True``: 32-bit columns stored as slab-relative 16-bit ones
        when they fit (core.slab_compress) -- 2 bytes less per nonzero."""
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.row_ptr = torch.as_tensor(np.asarray(row_ptr, dtype=np.int64)).to(torch.int32).to(dev)
        ci = np.asarray(col_idx)
        if ci.dtype not in (np.uint8, np.uint16, np.uint32):
            ci = ci.astype(np.uint32)
        # structure facts for the single-RHS stream kernel (csrc/stream.cu)
        self.band, self.blk_max = band_facts(row_ptr, ci)
        self.slab_base, self.slab_shift = None, 0
        if slab and ci.dtype == np.uint32:
            from .core import slab_compress
            sc = slab_compress(row_ptr, ci)
            if sc is not None:
                ci, base, self.slab_shift = sc
                self.slab_base = torch.from_numpy(base).to(dev)
        # 64 bytes of slack behind the entry arrays: the stream kernel fetches
        # stages in 16-byte units and may read past the last entry
        self.col_idx = _padded_to(ci, dev)
        self.values = _padded_to(np.asarray(values), dev)
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.nnz = int(self.col_idx.numel())
        # rows far longer than the mean run on whole CTAs (same bits)
        self.long_rows, self.long_thr = long_row_split(row_ptr, dev)

    @classmethod
    def from_block(cls, blk, device=None, slab=False):
        return cls(blk.row_ptr, blk.col_idx, blk.values, blk.nrows, blk.ncols, device, slab)

    def view(self) -> _lib.mrs_csr:
        v = _csr_view(self.row_ptr, self.col_idx, self.values, self.nrows, self.ncols)
        if self.slab_base is not None:
            v.slab_base = self.slab_base.data_ptr()
            v.slab_shift = self.slab_shift
        if self.long_rows is not None:
            v.long_rows = self.long_rows.data_ptr()
            v.n_long = int(self.long_rows.numel())
            v.long_thr = self.long_thr
        v.band, v.blk_max, v.flags = self.band, self.blk_max, 1
        return v


def _padded_to(arr, device):
    """Device copy of a 1-d host array as a view of an allocation with 64
    spare bytes behind it."""
    arr = np.ascontiguousarray(arr)
    t = torch.from_numpy(arr)
    extra = -(-64 // max(1, arr.itemsize))
    buf = torch.zeros(arr.size + extra, dtype=t.dtype, device=device)
    buf[:arr.size].copy_(t)
    return buf[:arr.size]


def band_facts(row_ptr, col_idx, block_rows=256):
    """(max |column - row|, most entries in an aligned block of ``block_rows``
    rows) of a CSR pattern, computed on the host in row blocks."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    n = rp.size - 1
    if n <= 0 or rp[-1] <= 0:
        return -1, 0
    ci = np.asarray(col_idx)
    band = 0
    step = 1 << 18
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        e0, e1 = int(rp[r0]), int(rp[r1])
        if e1 == e0:
            continue
        rows = np.repeat(np.arange(r0, r1, dtype=np.int64), np.diff(rp[r0:r1 + 1]))
        band = max(band, int(np.abs(ci[e0:e1].astype(np.int64) - rows).max()))
    edges = rp[np.minimum(np.arange(0, n + block_rows, block_rows), n)]
    blk_max = int(np.diff(edges).max())
    if band > 2 ** 30 or blk_max > 2 ** 30:
        return -1, 0
    return band, blk_max


def long_row_split(row_ptr, device):
    """Rows with more than max(64, 4 * ceil(mean)) entries, when they are
    outliers (at most 1/8 of the rows) -- the same rule as the solver's level
    upload (csrc/solver.cu upload_csr).  Returns (device int32 rows, thr) or
    (None, 0)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    n = rp.size - 1
    if n <= 0 or rp[-1] <= 0:
        return None, 0
    thr = max(64, 4 * (-(-int(rp[-1]) // n)))
    rows = np.flatnonzero(np.diff(rp) > thr).astype(np.int32)
    if rows.size == 0 or rows.size * 8 > n:
        return None, 0
    return torch.from_numpy(rows).to(device), thr


def _csr_view(row_ptr, col_idx, values, nrows, ncols):
    for t, nm in ((row_ptr, "row_ptr"), (col_idx, "col_idx"), (values, "values")):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous():
            raise InvalidArgumentError(f"{nm} must be a contiguous CUDA tensor")
    if row_ptr.dtype != torch.int32:
        raise InvalidArgumentError("device row_ptr must be int32 (see DeviceCsr)")
    if col_idx.dtype not in _IDX_BYTES or values.dtype not in _VAL_BYTES:
        raise InvalidArgumentError("unsupported index or value dtype")
    return _lib.mrs_csr(nrows, ncols, col_idx.numel(), row_ptr.data_ptr(), col_idx.data_ptr(),
                        values.data_ptr(), _IDX_BYTES[col_idx.dtype], _VAL_BYTES[values.dtype])


def csr_spmv(row_ptr, col_idx, values, x, y, mode, b=None):
    """y op= A x (_ckernels.pyx:30-57).  ``row_ptr`` may be a DeviceCsr, in which
    case ``col_idx``/``values`` are ignored.

    Extension: float32 block vectors (x, y and b all float32; the reference's
    are always float64) -- loads widened, float64 accumulation in entry order,
    one rounding at the store; m in {1, 2, 4, 8, 16, 32}."""
    if isinstance(row_ptr, DeviceCsr):
        view = row_ptr.view()
        ncols = row_ptr.ncols
    else:
        if row_ptr.dtype == torch.int64:
            row_ptr = row_ptr.to(torch.int32)
        ncols = x.shape[0]
        view = _csr_view(row_ptr, col_idx, values, row_ptr.numel() - 1, ncols)
    vdt = x.dtype if isinstance(x, torch.Tensor) and x.dtype == torch.float32 else torch.float64
    _vec(x, "x", vdt); _vec(y, "y", vdt)
    if mode not in (0, 1, 2, 3):
        raise ValueError(f"unknown spmv mode {mode}")
    if y.shape[0] != view.nrows or x.shape[1] != y.shape[1]:
        raise ShapeMismatchError(f"spmv shapes: A {view.nrows}x{ncols}, x {tuple(x.shape)}, "
                                 f"y {tuple(y.shape)}")
    if x.data_ptr() == y.data_ptr():
        raise InvalidArgumentError("spmv output must not alias the input")
    bp = None
    if mode == MODE_RSUB:
        _vec(b, "b", vdt)
        if b.shape != y.shape:
            raise ShapeMismatchError("b and y shapes differ")
        bp = b.data_ptr()
    fn = _lib.lib().mrs_csr_spmv if vdt == torch.float64 else _lib.lib().mrs_csr_spmv_f32
    _ck(fn(C.byref(view), x.data_ptr(), y.data_ptr(), x.shape[1], mode, bp, _stream()), "csr_spmv")


def _same(*ts):
    s = ts[0].shape
    for t in ts[1:]:
        if t.shape != s:
            raise ShapeMismatchError(f"block vector shapes differ: {tuple(s)} vs {tuple(t.shape)}")


def axpby(a, x, b, y):
    """y := a*x + b*y columnwise (_ckernels.pyx:82-89)."""
    _vec(x, "x"); _vec(y, "y"); _same(x, y)
    n, m = y.shape
    a, b = _scal(a, m, y.device), _scal(b, m, y.device)
    _ck(_lib.lib().mrs_axpby(n, m, a.data_ptr(), x.data_ptr(), b.data_ptr(), y.data_ptr(),
                             _stream()), "axpby")


def add2_scaled(y, a, u, b, v):
    """y := (y + a*u) + b*v (_ckernels.pyx:92-99)."""
    for t, nm in ((y, "y"), (u, "u"), (v, "v")):
        _vec(t, nm)
    _same(y, u, v)
    n, m = y.shape
    a, b = _scal(a, m, y.device), _scal(b, m, y.device)
    _ck(_lib.lib().mrs_add2_scaled(n, m, y.data_ptr(), a.data_ptr(), u.data_ptr(), b.data_ptr(),
                                   v.data_ptr(), _stream()), "add2_scaled")


def dot_partial(x, y):
    """Per-column inner products (_ckernels.pyx:102-111); (m,) CUDA tensor."""
    _vec(x, "x"); _vec(y, "y"); _same(x, y)
    n, m = x.shape
    out = torch.empty(m, dtype=torch.float64, device=x.device)
    _ck(_lib.lib().mrs_dot(n, m, x.data_ptr(), y.data_ptr(), out.data_ptr(), _stream()), "dot")
    return out


def fused_update_dot(a, x, b, y):
    """y := a*x + b*y; return dot(y, y) (_ckernels.pyx:114-127)."""
    _vec(x, "x"); _vec(y, "y"); _same(x, y)
    n, m = y.shape
    a, b = _scal(a, m, y.device), _scal(b, m, y.device)
    out = torch.empty(m, dtype=torch.float64, device=y.device)
    _ck(_lib.lib().mrs_fused_update_dot(n, m, a.data_ptr(), x.data_ptr(), b.data_ptr(),
                                        y.data_ptr(), out.data_ptr(), _stream()),
        "fused_update_dot")
    return out


def fused_paired_update(y1, a, u, b, s, y2, c, w):
    """y1 += a*u + b*s; y2 := s - c*w (_ckernels.pyx:130-142)."""
    for t, nm in ((y1, "y1"), (u, "u"), (s, "s"), (y2, "y2"), (w, "w")):
        _vec(t, nm)
    _same(y1, u, s, y2, w)
    n, m = y1.shape
    a, b, c = (_scal(t, m, y1.device) for t in (a, b, c))
    _ck(_lib.lib().mrs_fused_paired_update(n, m, y1.data_ptr(), a.data_ptr(), u.data_ptr(),
                                           b.data_ptr(), s.data_ptr(), y2.data_ptr(),
                                           c.data_ptr(), w.data_ptr(), _stream()),
        "fused_paired_update")


def fused_update_dot2(y, u, c, w, z):
    """y := u - c*w; return (dot(z, y), dot(y, y)) (_ckernels.pyx:145-162)."""
    for t, nm in ((y, "y"), (u, "u"), (w, "w"), (z, "z")):
        _vec(t, nm)
    _same(y, u, w, z)
    n, m = y.shape
    c = _scal(c, m, y.device)
    d1 = torch.empty(m, dtype=torch.float64, device=y.device)
    d2 = torch.empty(m, dtype=torch.float64, device=y.device)
    _ck(_lib.lib().mrs_fused_update_dot2(n, m, y.data_ptr(), u.data_ptr(), c.data_ptr(),
                                         w.data_ptr(), z.data_ptr(), d1.data_ptr(), d2.data_ptr(),
                                         _stream()), "fused_update_dot2")
    return d1, d2


def gs_sweep(row_ptr, col_idx, values, diag_pos, b, c, x, forward):
    """One Gauss-Seidel half-sweep in place on x (_ckernels.pyx:60-79):
    v = b - c, v -= a_ik x_k for k != diag_pos[i] in entry order, x_i = v / a_ii,
    rows ascending (``forward``) or descending -- bitwise the sequential
    sweep, run level by level on one thread-block cluster (csrc/sgs.cuh).
    ``row_ptr`` may be a DeviceCsr (``col_idx``/``values`` then ignored).

    Off the hot path: this plugin entry is SYNCHRONOUS and rebuilds the level
    schedule on the host from the device structure on every call (solver plans
    build theirs once at upload and replay it inside the solve graph)."""
    if isinstance(row_ptr, DeviceCsr):
        view = row_ptr.view()
    else:
        if row_ptr.dtype == torch.int64:
            row_ptr = row_ptr.to(torch.int32)
        view = _csr_view(row_ptr, col_idx, values, row_ptr.numel() - 1, row_ptr.numel() - 1)
    for t, nm in ((b, "b"), (c, "c"), (x, "x")):
        _vec(t, nm)
    _same(b, c, x)
    if x.shape[0] != view.nrows or view.nrows != view.ncols:
        raise ShapeMismatchError(f"gs_sweep: A {view.nrows}x{view.ncols}, x {tuple(x.shape)}")
    if not (isinstance(diag_pos, torch.Tensor) and diag_pos.is_cuda):
        raise InvalidArgumentError("diag_pos must be a CUDA tensor")
    dp = diag_pos.to(torch.int64).contiguous()
    if dp.numel() != view.nrows:
        raise ShapeMismatchError("diag_pos must have one entry per row")
    _ck(_lib.lib().mrs_gs_sweep(C.byref(view), dp.data_ptr(), b.data_ptr(), c.data_ptr(),
                                x.data_ptr(), x.shape[1], int(bool(forward)), _stream()),
        "gs_sweep")
