"""cProfile of prepare() for one bench configuration (setup-phase breakdown).

    python scripts/profile_prepare.py --config c4 [--grid 128]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--m", type=int, default=None)
    a = ap.parse_args()
    import torch  # noqa: F401  (import cost outside the profile)
    import bench
    from paper_2103_07329_b200.params import tree
    from paper_2103_07329_b200.solvers import prepare
    bench.select(a.config, a.grid)
    A = bench.make_matrix()
    torch.cuda.init()
    pr = cProfile.Profile()
    t0 = time.time()
    pr.enable()
    cs = prepare(tree(bench.ROLES), A)
    cs.plan_factory(a.m or bench.M)
    torch.cuda.synchronize()
    pr.disable()
    print(f"prepare + plan: {time.time() - t0:.2f} s  (n = {A.nrows}, nnz = {A.nnz})")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(35)


if __name__ == "__main__":
    main()
