"""Small solves that cover the hand-rolled synchronisation protocols, for
compute-sanitizer (racecheck / synccheck / memcheck, one tool per run):
  * last-CTA atomic-ticket reduction folds (every Krylov dot, fused epilogues);
  * the conditional-WHILE graph with device-set conditionals;
  * Gauss-Seidel half-sweeps on one thread-block cluster (cluster barriers,
    L1-coherent plain loads) and on one CTA;
  * long-row CTAs of the SpMM (shared-memory products), the dense DMMA tail;
  * the fp32-vector V-cycle and the plugin kernels.
    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2103_07329_b200 import BlockVector, gen_poisson3d, kernels as K  # noqa: E402
from paper_2103_07329_b200.io import gen_stencil27_aniso  # noqa: E402
from paper_2103_07329_b200.params import tree  # noqa: E402
from paper_2103_07329_b200.solvers import prepare  # noqa: E402

JAC = {"method": "Jacobi", "weight": "0.8"}
CHEB = {"method": "Chebyshev", "polynomial_order": "2"}
CASES = [
    ("c1_jacobi_pcg", gen_poisson3d(16, 16, 16)[0], 4,
     {"solver": {"method": "CG", "max_iters": "400"}, "preconditioner": {"method": "Jacobi"}}),
    ("c2_amg_pcg", gen_poisson3d(20, 20, 20)[0], 8,
     {"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"},
      "pre_smoother": JAC, "post_smoother": JAC}),
    ("c2g_amg_pcg_sgs", gen_poisson3d(12, 12, 12)[0], 8,
     {"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"}}),
    ("c3_amg_bicgstab_mixed", gen_poisson3d(16, 16, 16)[0], 16,
     {"solver": {"method": "BiCGStab"},
      "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": "1"},
      "pre_smoother": CHEB, "post_smoother": CHEB}),
    ("c3_vec32", gen_poisson3d(16, 16, 16)[0], 8,
     {"solver": {"method": "BiCGStab"},
      "preconditioner": {"method": "MultiGrid", "mg_vector_precision": "fp32"},
      "pre_smoother": CHEB, "post_smoother": CHEB}),
    ("c4_27pt_pbicgstab", gen_stencil27_aniso(12, seed=4), 4,
     {"solver": {"method": "PBiCGStab"}, "preconditioner": {"method": "MultiGrid"},
      "pre_smoother": JAC, "post_smoother": JAC}),
]


def main():
    torch.cuda.set_device(0)
    for name, A, m, roles in CASES:
        B = np.random.default_rng(1).uniform(-1, 1, (A.nrows, m))
        X = BlockVector.zeros(A.nrows, m)
        st = prepare(tree(roles), A).run(BlockVector.from_array(B), X)
        print(f"{name}: iterations {st.iterations}, converged {st.all_converged}", flush=True)
    # plugin kernels: SpMM over an operator with long rows (whole-CTA rows),
    # the ticketed dot reduction on two streams
    n = 3000
    rng = np.random.default_rng(2)
    dense = (rng.random((n, n)) < 0.004) * rng.standard_normal((n, n))
    dense[:8] = rng.standard_normal((8, n))                 # 8 rows of 3000 entries
    from paper_2103_07329_b200.core import CsrBlock
    blk = CsrBlock.from_dense(dense)
    D = K.DeviceCsr.from_block(blk)
    x = torch.rand(n, 8, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    K.csr_spmv(D, None, None, x, y, K.MODE_ASSIGN)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        d1 = K.dot_partial(x, y)
    with torch.cuda.stream(s2):
        d2 = K.dot_partial(y, x)
    torch.cuda.synchronize()
    print("plugin ok", float((d1 - d2).abs().max()))
