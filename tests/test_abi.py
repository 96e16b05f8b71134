"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares (no device calls here)."""

import ctypes
import os
import re

from paper_2103_07329_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mrsolve_b200.h")).read()
    return sorted(set(re.findall(r"\b(mrs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_status_strings_and_version():
    assert _lib.lib().mrs_version() >= 1
    assert _lib.status_string(0) == "ok"
    assert "breakdown" in _lib.status_string(5).lower()


def test_struct_layouts_match_header(tmp_path):
    """Compile a probe against the header and compare every struct's size and
    field offsets with the ctypes mirrors."""
    import subprocess
    structs = [_lib.mrs_csr, _lib.mrs_host_csr, _lib.mrs_smoother, _lib.mrs_plan_desc,
               _lib.mrs_stats, _lib.mrs_amg_params]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "mrsolve_b200.h"',
             'int main(void) {']
    for s in structs:
        lines.append(f'printf("{s.__name__} %zu\\n", sizeof({s.__name__}));')
        for f, _ in s._fields_:
            lines.append(f'printf("{s.__name__}.{f} %zu\\n", offsetof({s.__name__}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for s in structs:
        assert int(got[s.__name__]) == ctypes.sizeof(s), s.__name__
        for f, _ in s._fields_:
            assert int(got[f"{s.__name__}.{f}"]) == getattr(s, f).offset, f"{s.__name__}.{f}"


def test_plan_rejects_bad_descriptors_without_gpu():
    L = _lib.lib()
    d = _lib.mrs_plan_desc()
    d.m = 0
    d.nrows = 10
    h = ctypes.c_void_p()
    assert L.mrs_plan_create(ctypes.byref(d), ctypes.byref(h)) == _lib.MRS_ERR_ARG
    d.m = 4
    d.method = 7
    assert L.mrs_plan_create(ctypes.byref(d), ctypes.byref(h)) == _lib.MRS_ERR_UNSUPPORTED


def test_product_path_fails_loudly_without_the_extension(monkeypatch):
    """No CPU fallback: a missing library is an ImportError, not a slow path."""
    import pytest
    from paper_2103_07329_b200 import build
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIBPATH", "/nonexistent/libmrsolve_b200.so")
    monkeypatch.setattr(build, "needs_build", lambda: False)
    with pytest.raises(ImportError):
        _lib.lib()


def test_kernel_plugin_rejects_host_tensors():
    import numpy as np
    import pytest
    import torch
    from paper_2103_07329_b200 import kernels as K
    from paper_2103_07329_b200.errors import InvalidArgumentError
    x = torch.zeros(4, 2, dtype=torch.float64)
    with pytest.raises(InvalidArgumentError):
        K.axpby(1.0, x, 1.0, x.clone())
    with pytest.raises(InvalidArgumentError):
        K.dot_partial(x, x)


def test_reference_objects_are_accepted_by_duck_typing():
    """A reference CsrBlock / BlockVector (same attributes) converts without
    copying semantics changes (core.as_csr / as_block_vector)."""
    import numpy as np
    from paper_2103_07329_b200.core import as_block_vector, as_csr
    from paper_2103_07329_b200.io import gen_poisson3d

    class RefLike:                     # attribute contract of mrsolve.core.CsrBlock
        def __init__(self, b):
            self.nrows, self.ncols = b.nrows, b.ncols
            self.row_ptr, self.col_idx, self.values = b.row_ptr, b.col_idx, b.values

    A, b = gen_poisson3d(4, 3, 2)
    C = as_csr(RefLike(A))
    assert C.nrows == A.nrows and np.array_equal(C.values, A.values)
    assert as_block_vector(b) is b
