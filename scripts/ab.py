#!/usr/bin/env python
"""A/B a tuning knob inside ONE process (box-to-box variance is ~20%).

    python scripts/ab.py --knob pdl --values 0 1 --config c2 --rounds 3

Each round prepares a fresh solver per value (graphs are captured at the
first solve) and times `steps` solves with CUDA events, L2 flushed between.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--knob", default="spmm_staged")
    ap.add_argument("--values", type=int, nargs="+", default=[0, 1])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--grid", type=int, default=None)
    a = ap.parse_args()
    import numpy as np
    import torch
    import bench
    from paper_2103_07329_b200 import _lib, gen_poisson3d
    from paper_2103_07329_b200.params import tree
    from paper_2103_07329_b200.solvers import prepare
    bench.select(a.config, a.grid)
    A = bench.make_matrix()
    B = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (A.nrows, bench.M))).cuda()
    X = torch.zeros_like(B)
    flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
    sink = torch.empty((), dtype=torch.float64, device="cuda")
    res = {v: [] for v in a.values}
    iters = {}
    h = None
    for r in range(a.rounds):
        for v in a.values:
            if a.knob == "dense_tail_rows":        # setup-phase (Python) knob
                from paper_2103_07329_b200 import amg
                amg.set_dense_tail_rows(v)
            elif a.knob == "dense_bw":              # cost-model bandwidth (GB/s)
                from paper_2103_07329_b200 import amg
                amg._DENSE_BW = float(v) * 1e3
            else:
                _lib.set_option(a.knob, v)
            cs = prepare(tree(bench.ROLES), A, hierarchy=h)
            h = h or cs.hierarchy
            for _ in range(3):
                cs.run(B, X, x_is_zero=True)
            ts = []
            for _ in range(a.steps):
                torch.sum(flush, dim=0, out=sink)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); st = cs.run(B, X, x_is_zero=True); e1.record(); e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[v].append(sorted(ts)[len(ts) // 2])
            iters[v] = st.iterations
            del cs
    for v in a.values:
        print(f"{a.knob}={v}: median ms/solve per round {['%.3f' % t for t in res[v]]}  "
              f"best {min(res[v]):.3f}  iters {iters[v]}")


if __name__ == "__main__":
    main()
