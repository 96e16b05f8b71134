#!/usr/bin/env python
"""Warm per-launch device times of one solver iteration (CUDA events around
each launch; no profiler).  Complements the cold ncu launch list.

    python scripts/warm_profile.py --config c2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    import numpy as np
    import torch
    import bench
    from paper_2103_07329_b200 import gen_poisson3d
    from paper_2103_07329_b200.params import tree
    from paper_2103_07329_b200.solvers import prepare
    bench.select(a.config)
    A = bench.make_matrix()
    B = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (A.nrows, bench.M))).cuda()
    X = torch.zeros_like(B)
    cs = prepare(tree(bench.ROLES), A)
    cs.run(B, X, x_is_zero=True)
    plan = cs.plan_factory(bench.M)
    t = plan.profile(3, B)
    t = plan.profile(3, B)
    import re
    vec_ops = ["axpby", "add2", "paired", "dot", "update_dot", "update_dot2", "copy",
               "cg_update", "cg_update_jac", "p_update", "seed", "bicg_p", "bicg_s", "dot3",
               "bicg_xr", "dot2", "dot5", "bicg_xr0", "pbicg_qy", "pbicg_w"]
    sp_ops = ["SPMV", "JAC_SWEEP", "CHEB_FIRST", "CHEB_STEP"]
    names = []
    for nm in plan.launch_names():
        mv = re.search(r"vec_kernel<(\d+)>", nm)
        ms = re.search(r"spmm_kernel<(\d+), (\d), ([a-z ]+), ([a-z ]+)>", nm)
        if mv:
            nm = f"vec {vec_ops[int(mv.group(1))]}"
        elif ms:
            nm = f"spmm m={ms.group(1)} {sp_ops[int(ms.group(2))]} {ms.group(3)} {ms.group(4)}"
        names.append(nm)
    print(f"{len(t)} launches/iteration, sum {t.sum():.1f} us")
    for i, v in enumerate(t):
        nm = names[i] if i < len(names) else ""
        nm = nm.replace("mrs::", "").replace("unsigned ", "u")
        print(f"{i:3d} {v:8.2f}  {nm[:110]}")


if __name__ == "__main__":
    main()
