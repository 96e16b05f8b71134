#!/usr/bin/env python
"""Micro-benchmark of one SpMM launch configuration (for ncu captures).

    python scripts/spmm_micro.py --matrix c2 --m 8 --mode rsub --reps 20
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--matrix", default="c2", choices=["c2", "c3", "c4", "c5", "c2l1", "c3l1"])
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--mode", default="rsub", choices=["assign", "rsub"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--no-slab", action="store_true", help="plain 32-bit columns")
    ap.add_argument("--knob", action="append", default=[], help="name=value (mrs_set_option)")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2103_07329_b200 import _lib
    for kv in a.knob:
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    from paper_2103_07329_b200 import gen_poisson3d, gen_random_sdd, kernels as K
    if a.matrix == "c5":
        A = gen_random_sdd()
    elif a.matrix == "c4":
        from paper_2103_07329_b200 import gen_stencil27_aniso
        A = gen_stencil27_aniso(128, seed=4)
    elif a.matrix == "c2l1":
        from paper_2103_07329_b200.amg import setup
        A = setup(gen_poisson3d(64, 64, 64)[0]).levels[1].A
    elif a.matrix == "c3l1":          # C3's level 1 (mixed precision: f32 values)
        from paper_2103_07329_b200.amg import setup
        A = setup(gen_poisson3d(128, 128, 128)[0], mixed_precision=True).levels[1].A
    else:
        g = 64 if a.matrix == "c2" else 128
        A = gen_poisson3d(g, g, g)[0]
    vals = A.values.astype(np.float32) if a.f32 else A.values
    D = K.DeviceCsr(A.row_ptr, A.col_idx, vals, A.nrows, A.ncols, slab=not a.no_slab)
    x = torch.rand(A.ncols, a.m, dtype=torch.float64, device="cuda")
    b = torch.rand(A.nrows, a.m, dtype=torch.float64, device="cuda")
    y = torch.empty_like(b)
    mode = K.MODE_RSUB if a.mode == "rsub" else K.MODE_ASSIGN
    flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
    sink = torch.empty((), dtype=torch.float64, device="cuda")
    ts = []
    for r in range(a.reps):
        torch.sum(flush, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K.csr_spmv(D, None, None, x, y, mode, b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    t = sorted(ts)[len(ts) // 2]
    vb = vals.itemsize
    nslab = 0 if D.slab_base is None else D.slab_base.numel()
    byts = (A.nnz * (vb + D.col_idx.element_size()) + (A.nrows + 1) * 4 + 4 * nslab
            + (A.ncols + A.nrows * (2 if mode else 1)) * a.m * 8)
    print(f"{a.matrix} n={A.nrows} nnz={A.nnz} m={a.m} {a.mode} idx={'u16slab' if nslab else 'u' + str(8 * D.col_idx.element_size())}: {t:.2f} us (L2 flushed), "
          f"{byts / t / 1e3:.0f} GB/s algorithmic")


if __name__ == "__main__":
    main()
