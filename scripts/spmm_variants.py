"""A/B of the SpMM variants (lane / cooperative loads / 16 in flight) on the
BASELINE operators: C5 (random banded SDD, n = 2^22), the C2 / C3 fine 7-point
operators and the C4 27-point operator at 128^3; every m of the C5 sweep.
Each point: median of 9 single launches after an L2 flush (ASSIGN mode), and
what the per-operator autotune (plugin path) picked.

    python scripts/spmm_variants.py [--quick] > gpurun_out/spmm_variants.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2103_07329_b200 import _lib, gen_poisson3d, kernels as K  # noqa: E402
from paper_2103_07329_b200.io import gen_random_sdd, gen_stencil27_aniso  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
sink = torch.empty((), dtype=torch.float64, device="cuda")


def timed(D, x, y, reps=9):
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K.csr_spmv(D, None, None, x, y, K.MODE_ASSIGN)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return sorted(ts)[reps // 2]


def main():
    quick = "--quick" in sys.argv
    mats = {"c5": gen_random_sdd(), "c2_64": gen_poisson3d(64, 64, 64)[0],
            "p7_128": gen_poisson3d(128, 128, 128)[0], "c4_128": gen_stencil27_aniso(128, seed=4)}
    out = []
    for name, A in mats.items():
        for vdt in ("f64", "f32"):
            vals = A.values if vdt == "f64" else A.values.astype(np.float32)
            for slab in (False, True):
                if name != "c5" and not slab:
                    continue
                if name != "c5" and vdt == "f32":
                    continue
                D = K.DeviceCsr(A.row_ptr, A.col_idx, vals, A.nrows, A.ncols, slab=slab)
                ib = D.col_idx.element_size()
                nslab = 0 if D.slab_base is None else D.slab_base.numel()
                for m in ([8] if quick else [1, 2, 4, 8, 16, 32]):
                    x = torch.rand(A.ncols, m, dtype=torch.float64, device="cuda")
                    y = torch.empty(A.nrows, m, dtype=torch.float64, device="cuda")
                    byts = (A.nnz * (vals.itemsize + ib) + (A.nrows + 1) * 4 + 4 * nslab
                            + 2 * A.nrows * m * 8)
                    row = {"op": name, "values": vdt, "idx": "u16slab" if nslab else f"u{8*ib}",
                           "m": m, "bytes": byts}
                    only = os.environ.get("VARIANTS")      # e.g. VARIANTS=lane,pair
                    for v, vn in ((1, "lane"), (2, "coop"), (3, "long"), (4, "l2"), (5, "na"),
                                  (7, "pair")):
                        if only and vn not in only.split(","):
                            continue
                        if v == 2 and m not in (4, 8, 16):
                            continue
                        if v in (3, 4, 5) and m > 16:
                            continue
                        if v == 7 and m not in (2, 4, 8, 16):
                            continue
                        _lib.set_option("spmm_variant", v)
                        t = timed(D, x, y)
                        row[vn + "_us"] = t * 1e6
                        row[vn + "_frac"] = byts / t / 1e9 / PEAK
                    _lib.set_option("spmm_variant", 0)
                    t = timed(D, x, y)          # first call tunes (plugin cache)
                    row["auto_us"] = t * 1e6
                    row["auto_frac"] = byts / t / 1e9 / PEAK
                    out.append(row)
                    print(json.dumps(row), file=sys.stderr, flush=True)
                    del x, y
                del D
    print(json.dumps({"peak_gbs": PEAK, "points": out}))


if __name__ == "__main__":
    main()
