"""Fine-level 7-point SpMM (RSUB, slab) timing: sustained (graph of back-to-back
launches over 3 cold copies).  python scripts/p7_time.py GRID M"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2103_07329_b200 import gen_poisson3d, kernels as K
g, m = int(sys.argv[1]), int(sys.argv[2])
A = gen_poisson3d(g, g, g)[0]
sets = []
for _ in range(3):
    D = K.DeviceCsr.from_block(A, slab=True)
    x = torch.rand(A.ncols, m, dtype=torch.float64, device="cuda")
    b = torch.rand(A.nrows, m, dtype=torch.float64, device="cuda")
    sets.append((D, x, b, torch.empty_like(b)))
for (D, x, b, y) in sets:
    K.csr_spmv(D, None, None, x, y, K.MODE_RSUB, b)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    for _ in range(4):
        for (D, x, b, y) in sets:
            K.csr_spmv(D, None, None, x, y, K.MODE_RSUB, b)
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / 12)
print(f"g={g} m={m} sustained_us={sorted(ts)[3]:.2f}")
