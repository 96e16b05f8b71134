"""One product of the C5 operator (n = 2^22) at m = 1 through the plugin with the
stream kernel forced -- the command profiled for profiles/r02_stream_ncu.txt:

    python scripts/ncu_stream.py && ncu --set full --clock-control none --import-source on \
        -k regex:stream_spmv -c 1 -o gpurun_out/stream python scripts/ncu_stream.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07329_b200 import _lib, kernels as K  # noqa: E402
from paper_2103_07329_b200.io import gen_random_sdd  # noqa: E402

A = gen_random_sdd()
D = K.DeviceCsr(A.row_ptr, A.col_idx, A.values, A.nrows, A.ncols)
x = torch.rand(A.ncols, 1, dtype=torch.float64, device="cuda")
y = torch.empty(A.nrows, 1, dtype=torch.float64, device="cuda")
_lib.set_option("spmm_variant", 6)
for _ in range(3):
    K.csr_spmv(D, None, None, x, y, K.MODE_ASSIGN)
torch.cuda.synchronize()
print("stream launches", _lib.lib().mrs_stream_launches(), "band", D.band, "blk_max", D.blk_max)
