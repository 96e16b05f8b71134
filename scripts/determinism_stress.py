"""Race / synchronisation evidence without compute-sanitizer (closed on this
pool): every hand-rolled protocol must give the SAME bits on every repeat.

  * whole solves (ticket-folded dots + device epilogues + conditional-WHILE
    graph; Gauss-Seidel cluster / single-CTA sweeps; long-row CTAs; fp32
    V-cycle) repeated N times: X bitwise identical across repeats;
  * plugin dots on two concurrent streams (per-stream scratch): bitwise equal
    to the single-stream result, 1e-13 of the oracle;
Run with the checked library (device asserts on tickets / indices) too:
  MRS_LIB=paper_2103_07329_b200/libmrsolve_b200_checked.so python scripts/determinism_stress.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2103_07329_b200 import gen_poisson3d, kernels as K  # noqa: E402
from paper_2103_07329_b200.io import gen_stencil27_aniso  # noqa: E402
from paper_2103_07329_b200.params import tree  # noqa: E402
from paper_2103_07329_b200.solvers import prepare  # noqa: E402

JAC = {"method": "Jacobi", "weight": "0.8"}
CHEB = {"method": "Chebyshev", "polynomial_order": "2"}
CASES = [
    ("c1_jacobi_pcg", gen_poisson3d(24, 24, 24)[0], 4, 30,
     {"solver": {"method": "CG", "max_iters": "400"}, "preconditioner": {"method": "Jacobi"}}),
    ("c2_amg_pcg", gen_poisson3d(32, 32, 32)[0], 8, 30,
     {"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"},
      "pre_smoother": JAC, "post_smoother": JAC}),
    ("c2g_amg_pcg_sgs", gen_poisson3d(16, 16, 16)[0], 8, 10,
     {"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"}}),
    ("c3_amg_bicgstab_mixed", gen_poisson3d(24, 24, 24)[0], 16, 20,
     {"solver": {"method": "BiCGStab"},
      "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": "1"},
      "pre_smoother": CHEB, "post_smoother": CHEB}),
    ("c3_vec32_rbicgstab", gen_poisson3d(24, 24, 24)[0], 8, 20,
     {"solver": {"method": "RBiCGStab"},
      "preconditioner": {"method": "MultiGrid", "mg_vector_precision": "fp32"},
      "pre_smoother": CHEB, "post_smoother": CHEB}),
    ("c4_27pt_pbicgstab", gen_stencil27_aniso(20, seed=4), 4, 20,
     {"solver": {"method": "PBiCGStab"}, "preconditioner": {"method": "MultiGrid"},
      "pre_smoother": JAC, "post_smoother": JAC}),
]


def main():
    torch.cuda.set_device(0)
    bad = 0
    for name, A, m, reps, roles in CASES:
        B = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (A.nrows, m))).cuda()
        cs = prepare(tree(roles), A)
        ref = None
        same = 0
        for _ in range(reps):
            X = torch.zeros_like(B)
            st = cs.run(B, X, x_is_zero=True)
            Xh = X.cpu().numpy()
            if ref is None:
                ref = (Xh, st.iterations)
            same += int(np.array_equal(Xh, ref[0]) and st.iterations == ref[1])
        ok = same == reps and st.all_converged
        bad += not ok
        print(f"{name}: {reps} solves, {same} bitwise identical, iterations {ref[1]}, "
              f"{'OK' if ok else 'MISMATCH'}", flush=True)
    # plugin dots: two concurrent streams, random shapes
    rng = np.random.default_rng(3)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    agree = 0
    rounds = 100
    for r in range(rounds):
        n, m = int(rng.integers(1, 400000)), int(rng.choice([1, 2, 4, 8, 16]))
        x = torch.from_numpy(rng.standard_normal((n, m))).cuda()
        y = torch.from_numpy(rng.standard_normal((n, m))).cuda()
        base = K.dot_partial(x, y).cpu().numpy()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            d1 = K.dot_partial(x, y)
        with torch.cuda.stream(s2):
            d2 = K.dot_partial(x, y)
        torch.cuda.synchronize()
        o = O.dot_partial(x.cpu().numpy(), y.cpu().numpy())
        close = np.allclose(base, o, rtol=1e-12, atol=1e-12 * np.abs(o).max())
        agree += int(np.array_equal(d1.cpu().numpy(), base) and
                     np.array_equal(d2.cpu().numpy(), base) and close)
    bad += agree != rounds
    print(f"plugin dots: {rounds} rounds on two concurrent streams, {agree} bitwise equal to "
          f"the single-stream result and within 1e-12 of the oracle", flush=True)
    print("ALL OK" if not bad else f"{bad} FAILURES")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
