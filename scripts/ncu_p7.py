"""One fine-level 7-point SpMM (RSUB, slab indices) for an ncu capture:
    python scripts/ncu_p7.py GRID M"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2103_07329_b200 import gen_poisson3d, kernels as K
g, m = int(sys.argv[1]), int(sys.argv[2])
A = gen_poisson3d(g, g, g)[0]
D = K.DeviceCsr.from_block(A, slab=True)
x = torch.rand(A.ncols, m, dtype=torch.float64, device="cuda")
b = torch.rand(A.nrows, m, dtype=torch.float64, device="cuda")
y = torch.empty_like(b)
for _ in range(3):
    K.csr_spmv(D, None, None, x, y, K.MODE_RSUB, b)
torch.cuda.synchronize()
print("ok")
