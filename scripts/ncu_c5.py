"""One C5 SpMM (n = 2^22, ASSIGN) per variant for an ncu capture:
    ncu --set full -k regex:spmm_kernel python scripts/ncu_c5.py M VARIANT [VALUES] [IDX] [VECTORS]
VALUES f64|f32, IDX u32|u16slab, VECTORS f64|f32"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2103_07329_b200 import _lib, kernels as K
from paper_2103_07329_b200.io import gen_random_sdd
m, variant = int(sys.argv[1]), int(sys.argv[2])
vdt = sys.argv[3] if len(sys.argv) > 3 else "f64"
A = gen_random_sdd()
vals = A.values if vdt == "f64" else A.values.astype(np.float32)
idx = sys.argv[4] if len(sys.argv) > 4 else "u32"
tdt = torch.float32 if len(sys.argv) > 5 and sys.argv[5] == "f32" else torch.float64
D = K.DeviceCsr(A.row_ptr, A.col_idx, vals, A.nrows, A.ncols, slab=idx == "u16slab")
x = torch.rand(A.ncols, m, dtype=tdt, device="cuda")
y = torch.empty(A.nrows, m, dtype=tdt, device="cuda")
_lib.set_option("spmm_variant", variant)
for _ in range(2):
    K.csr_spmv(D, None, None, x, y, K.MODE_ASSIGN)
torch.cuda.synchronize()
print("ok")
