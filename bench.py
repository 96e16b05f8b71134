#!/usr/bin/env python
"""Benchmark: AMG-PCG RHS*iterations/s on BASELINE.json config 2, plus the
blocked-SpMM HBM roofline (config 5 sweep).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (N=1): 64^3 7-point Poisson (reference generator), m = 8 seeded
uniform[-1,1] right-hand sides, zero initial guess, classical RS AMG V(1,1)
with weighted Jacobi (w = 0.8) preconditioning CG, fp64, tol 1e-8.  A step
is one whole solve with B, X resident in HBM; setup (prepare) is excluded,
like the reference's bench (src/cli.py:111-146).  L2 is flushed (256 MB read
) between timed steps, outside the per-step CUDA events.

N > 1 (torchrun): the one global system is row-partitioned over the ranks
(team.py: halo exchange + m-wide dot allreduce over NCCL, coarse levels
agglomerated) -- strong scaling; value = RHS*it/s of the whole job, timed as
the max over ranks.

--impl reference: the reference's own CPU implementation (oracle/_ref,
mrsolve with its Cython kernels) on this host, same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AMG-PCG RHS·iterations/sec; blocked SpMM HBM GB/s vs roofline"
UNIT = "RHS*it/s"
SEED, TOL = 0, 1e-8
#: shared by both arms' `config` (the driver compares the two key for key)
L2_NOTE = ("GPU arm: L2 flushed (256 MB read) between timed steps, outside the CUDA events; "
           "reference arm: host CPU, no GPU caches involved")
_JAC = {"method": "Jacobi", "weight": "0.8"}
_CHEB = {"method": "Chebyshev", "polynomial_order": "2"}
#: BASELINE.json configs on the reference generator (C4: builder-defined 27-pt)
CONFIGS = {
    "c1": dict(grid=32, m=4, workload=(
        "C1: 3D Poisson 7-pt 32^3 (n=32768), m=4 seeded uniform[-1,1] RHS, zero guess, "
        "Jacobi-preconditioned CG, fp64, tol 1e-8"),
        roles={"solver": {"method": "CG", "rel_tolerance": "1e-8", "max_iters": "1000"},
               "preconditioner": {"method": "Jacobi"}}),
    "c2": dict(grid=64, m=8, workload=(
        "C2: 3D Poisson 7-pt 64^3 (n=262144), m=8 seeded uniform[-1,1] RHS, zero guess, "
        "classical RS AMG V(1,1) weighted-Jacobi (w=0.8) + PCG, fp64, tol 1e-8"),
        roles={"solver": {"method": "CG", "rel_tolerance": "1e-8"},
               "preconditioner": {"method": "MultiGrid"},
               "pre_smoother": _JAC, "post_smoother": _JAC}),
    "c3": dict(grid=128, m=16, workload=(
        "C3: 3D Poisson 7-pt 128^3 (n=2097152), m=16 seeded uniform[-1,1] RHS, zero guess, "
        "classical RS AMG V(1,1) Chebyshev-2 + BiCGStab, mixed precision (fp32 hierarchy "
        "levels >= 1, fp64 vectors), tol 1e-8"),
        roles={"solver": {"method": "BiCGStab", "rel_tolerance": "1e-8"},
               "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": "1"},
               "pre_smoother": _CHEB, "post_smoother": _CHEB}),
    # C4 is specified at 256^3 on 8 GPUs (~450M nnz); the default here is the
    # same operator family at 128^3 (56M nnz) -- --grid 256 for the full size
    "c4": dict(grid=128, m=8, kind="s27", workload=(
        "C4: 3D anisotropic variable-coefficient 27-point SPD operator (coefficients "
        "log-uniform [1e-2,1e2] per cell, z-anisotropy 100:1, default_rng(4)), m=8 seeded RHS, "
        "zero guess, classical RS AMG V(1,1) weighted-Jacobi (w=0.8) + PCG, fp64, tol 1e-8"),
        roles={"solver": {"method": "CG", "rel_tolerance": "1e-8"},
               "preconditioner": {"method": "MultiGrid"},
               "pre_smoother": _JAC, "post_smoother": _JAC}),
}
# the same C3 problem through the reordered / pipelined formulations
# and the paper's Fig. 3 solver (PBiCGStab + AMG with
# aggressive coarsening on two levels, tests/test_acceptance.py:206-214)
for _v in ("RBiCGStab", "PBiCGStab"):
    _c = dict(CONFIGS["c3"])
    _c["roles"] = dict(_c["roles"], solver={"method": _v, "rel_tolerance": "1e-8"})
    _c["workload"] = _c["workload"].replace("+ BiCGStab", f"+ {_v}")
    CONFIGS["c3" + _v[0].lower()] = _c
# C2 with the reference's DEFAULT MultiGrid smoother (one symmetric hybrid
# Gauss-Seidel sweep, exact sequential order by level scheduling)
CONFIGS["c2g"] = dict(CONFIGS["c2"], workload=(
    "C2 system (3D Poisson 7-pt 64^3, m=8 seeded RHS, zero guess) with the reference-default "
    "MultiGrid smoother: RS AMG V(1,1) symmetric Gauss-Seidel + PCG, fp64, tol 1e-8"),
    roles={"solver": {"method": "CG", "rel_tolerance": "1e-8"},
           "preconditioner": {"method": "MultiGrid"}})
# C3 with the fp32-vector V-cycle (extension: "fp32 preconditioner"; levels
# 1 .. tail-1 store their block vectors in float32, fp64 accumulation)
CONFIGS["c3v32"] = dict(CONFIGS["c3"], workload=CONFIGS["c3"]["workload"].replace(
    "fp64 vectors)", "fp64 Krylov vectors, fp32 V-cycle vectors below level 0)"),
    roles=dict(CONFIGS["c3"]["roles"], preconditioner={
        "method": "MultiGrid", "mg_mixed_precision": "1", "mg_vector_precision": "fp32"}))
CONFIGS["c3v32a"] = dict(CONFIGS["c3"], workload=CONFIGS["c3"]["workload"].replace(
    "fp64 vectors)", "fp64 Krylov vectors, fp32 V-cycle vectors on every level incl. 0)"),
    roles=dict(CONFIGS["c3"]["roles"], preconditioner={
        "method": "MultiGrid", "mg_mixed_precision": "1", "mg_vector_precision": "fp32_all"}))
CONFIGS["c4v32a"] = dict(CONFIGS["c4"], workload=CONFIGS["c4"]["workload"].replace(
    "fp64, tol", "fp64 Krylov vectors, fp32 V-cycle vectors on every level incl. 0, tol"),
    roles=dict(CONFIGS["c4"]["roles"], preconditioner={
        "method": "MultiGrid", "mg_vector_precision": "fp32_all"}))
CONFIGS["c2v32"] = dict(CONFIGS["c2"], workload=CONFIGS["c2"]["workload"].replace(
    "fp64, tol", "fp64 Krylov vectors, fp32 V-cycle vectors below level 0, tol"),
    roles=dict(CONFIGS["c2"]["roles"], preconditioner={
        "method": "MultiGrid", "mg_vector_precision": "fp32"}))
CONFIGS["fig3"] = dict(grid=128, m=16, workload=(
    "Fig. 3 solver on 3D Poisson 7-pt 128^3, m=16 seeded RHS, zero guess: PBiCGStab + RS AMG "
    "(aggressive coarsening on 2 levels, 2 paths, coarse <= 500) V(1,1) Chebyshev-2, fp64, "
    "tol 1e-8"),
    roles={"solver": {"method": "PBiCGStab", "rel_tolerance": "1e-8"},
           "preconditioner": {"method": "MultiGrid", "mg_agg_num_levels": "2",
                              "mg_coarse_matrix_size": "500", "mg_num_paths": "2"},
           "pre_smoother": _CHEB, "post_smoother": _CHEB})
CFG = CONFIGS["c2"]
GRID, M = CFG["grid"], CFG["m"]
WORKLOAD, ROLES = CFG["workload"], CFG["roles"]
REF_SNIPPET = r"""
import json, sys, time, numpy as np
import mrsolve
from mrsolve.core import BlockVector, CsrBlock
from mrsolve.io import gen_poisson3d
grid, m, seed, tol, steps, warmup = {grid}, {m}, {seed}, {tol}, {steps}, {warmup}
col0, ncol, nproc, bdir = {col0}, {ncol}, {nproc}, {bdir!r}
roles = {roles}
if {s27}:       # builder-defined C4 operator (not in the reference): our generator
    sys.path.insert(0, {root!r})
    from paper_2103_07329_b200.io import gen_stencil27_aniso
    G = gen_stencil27_aniso(grid, seed=4)
    A = CsrBlock(G.nrows, G.ncols, G.row_ptr, G.col_idx, G.values)
else:
    A, _ = gen_poisson3d(grid, grid, grid)
B = np.random.default_rng(seed).uniform(-1.0, 1.0, (A.nrows, m))[:, col0:col0 + ncol].copy()
t = mrsolve.ParamTree()
for role, e in roles.items():
    t.add_map(role, e)
t.set_defaults()
t0 = time.perf_counter()
cs = mrsolve.prepare(t, A)
setup = time.perf_counter() - t0
out = []
for k in range(warmup + steps):
    if k == warmup and nproc > 1:      # all processes start their timed solves together
        import os
        open(os.path.join(bdir, "ready_%d" % col0), "w").close()
        t0 = time.time()
        while len([f for f in os.listdir(bdir) if f.startswith("ready_")]) < nproc:
            if time.time() - t0 > 600:
                break
            time.sleep(0.005)
    X = BlockVector.zeros(A.nrows, ncol)
    t0 = time.perf_counter()
    st = cs.run(BlockVector.from_array(B), X)
    dt = time.perf_counter() - t0
    if k >= warmup:
        out.append((dt, st.iterations, float(st.final_rel_residual.max())))
print("REFJSON" + json.dumps(dict(setup=setup, runs=out, backend=mrsolve.kernels.BACKEND)))
"""


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-spmm", action="store_true", help="skip the config-5 SpMM sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--quick", action="store_true", help="small SpMM sweep (m=8 only)")
    ap.add_argument("--grid", type=int, default=None, help="override the config's grid size")
    ap.add_argument("--team", action="store_true",
                    help="use the row-partitioned (NCCL) path even with one rank")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS),
                    help="workload (default c2, the BASELINE metric's configuration)")
    ap.add_argument("--exec", default="graph", choices=["graph", "eager"],
                    help="eager: per-kernel launches (ncu cannot profile kernels inside "
                         "graphs with conditional nodes)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------

REASONS = [("gpu_idle", 0x1), ("applications_clocks_setting", 0x2), ("sw_power_cap", 0x4),
           ("hw_slowdown", 0x8), ("sync_boost", 0x10), ("sw_thermal_slowdown", 0x20),
           ("hw_thermal_slowdown", 0x40), ("hw_power_brake_slowdown", 0x80),
           ("display_clock_setting", 0x100)]


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 3:
                    try:
                        rows.append((float(p[0]), float(p[1]), int(p[2], 16)))
                    except ValueError:
                        pass
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = sorted(r[0] for r in rows)
        mask = 0
        for r in rows:
            mask |= r[2]
        reasons = [nm for nm, bit in REASONS if mask & bit and nm != "gpu_idle"]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# reference arm / cpu baseline
# ---------------------------------------------------------------------------

def run_reference_cpu(steps: int, warmup: int, timeout: float = 900.0, nproc: int = 1):
    """Run the reference (oracle/_ref: mrsolve + its Cython kernels) on this
    host's CPU.  Its kernels hold the GIL, so a process uses one core; with
    nproc > 1 the RHS columns are split over nproc processes, each pinned to
    its own core, started together after their setup (the reference's own
    solver on every usable host core).  Returns per-step (max wall time over
    the processes, sum of column*iterations) plus setup / backend."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "mrsolve")):
        return None, "oracle/_ref missing (run oracle/build_ref.sh)"
    env = dict(os.environ, PYTHONPATH=ref, MRSOLVE_KERNELS="cython", OMP_NUM_THREADS="1",
               OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    try:
        cores = sorted(os.sched_getaffinity(0))
    except Exception:
        cores = list(range(os.cpu_count() or 1))
    nproc = max(1, min(nproc, M, len(cores)))
    bdir = tempfile.mkdtemp(prefix="mrs_refbar_")
    cols = [(M * i // nproc, M * (i + 1) // nproc) for i in range(nproc)]
    procs = []
    for i, (c0, c1) in enumerate(cols):
        # the reference knows no fp32-vector V-cycle (our extension): its arm
        # runs the same configuration with fp64 vectors
        ref_roles = {r: {k: v for k, v in e.items() if k != "mg_vector_precision"}
                     for r, e in ROLES.items()}
        code = REF_SNIPPET.format(grid=GRID, m=M, seed=SEED, tol=TOL, steps=steps, warmup=warmup,
                                  roles=repr(ref_roles), s27=CFG.get("kind") == "s27", root=ROOT,
                                  col0=c0, ncol=c1 - c0, nproc=nproc, bdir=bdir)
        cmd = ["taskset", "-c", str(cores[i % len(cores)]), sys.executable, "-c", code]
        procs.append(subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    results, err = [], None
    for pr in procs:
        try:
            o, e = pr.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            pr.kill()
            o, e = pr.communicate()
        got = [json.loads(l[7:]) for l in o.splitlines() if l.startswith("REFJSON")]
        if not got:
            err = (e or o)[-400:]
        else:
            results.append(got[0])
    import shutil
    shutil.rmtree(bdir, ignore_errors=True)
    if err or len(results) != nproc:
        return None, err
    nsteps = min(len(r["runs"]) for r in results)
    runs = []
    for k in range(nsteps):
        dt = max(r["runs"][k][0] for r in results)
        work = sum((c1 - c0) * r["runs"][k][1] for (c0, c1), r in zip(cols, results))
        its = max(r["runs"][k][1] for r in results)
        runs.append((dt, work, its))
    return dict(setup=max(r["setup"] for r in results), runs=runs, nproc=nproc,
                backend=results[0]["backend"]), None


def reference_arm(args, rank):
    if rank != 0:
        return
    ncores = os.cpu_count()
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = ncores or 1
    # The reference's kernels hold the GIL (one core per process).  Two ways to
    # put the host's cores on the one solve: one process with all m columns,
    # or the columns split over min(m, cores) concurrent processes.  Its cost
    # per iteration is mostly column-independent, so the split rarely wins;
    # both are measured and the faster one is the reported baseline.
    tried = {}
    for nproc in sorted({1, min(M, usable)}):
        res, err = run_reference_cpu(args.steps, args.warmup, nproc=nproc)
        if res is not None:
            runs = res["runs"]
            tried[res["nproc"]] = (sum(r[1] for r in runs) / sum(r[0] for r in runs), res)
    if not tried:
        print(json.dumps({"impl": "reference", "unavailable": f"reference CPU run failed: {err}"}))
        return
    P = max(tried, key=lambda k: tried[k][0])
    val, res = tried[P]
    runs = res["runs"]
    tot = sum(r[0] for r in runs)
    its = [r[2] for r in runs]
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(runs), "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(runs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference gen_poisson3d + default_rng(0).uniform(-1,1) RHS",
        "config": {"workload": WORKLOAD, "n": GRID ** 3, "m": M, "iterations": its[0],
                   "l2": L2_NOTE},
        "details": {"parallelism": (f"{P} process(es) x 1 core, the m RHS columns split over "
                                    "them (reference kernels hold the GIL: one core per "
                                    "process)"),
                    "tried": {f"{k}_process": v[0] for k, v in sorted(tried.items())},
                    "setup_s_excluded": res["setup"]},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": P, "kind": "reference",
                         "sample": f"{len(runs)} full {args.config.upper()} solves after "
                                   f"{args.warmup} warm-up, m={M} columns over {P} concurrent "
                                   f"single-core process(es) ({P} of {ncores} host cores; the "
                                   f"faster of 1 and {min(M, usable)} processes), "
                                   f"mrsolve backend {res['backend']}; step time = the slowest "
                                   f"process"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def roofline_at_scale(torch, K, peak, grid=128):
    from paper_2103_07329_b200 import gen_poisson3d
    A = gen_poisson3d(grid, grid, grid)[0]
    D = K.DeviceCsr.from_block(A, slab=True)
    n = A.nrows
    x = torch.rand(n, M, dtype=torch.float64, device="cuda")
    b = torch.rand(n, M, dtype=torch.float64, device="cuda")
    y = torch.empty_like(b)
    for _ in range(3):
        K.csr_spmv(D, None, None, x, y, K.MODE_RSUB, b)
    reps, ts = 20, []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _r in range(reps):
            K.csr_spmv(D, None, None, x, y, K.MODE_RSUB, b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / reps)
    t = sorted(ts)[1]
    nslab = 0 if D.slab_base is None else D.slab_base.numel()
    byts = (A.nnz * (A.values.itemsize + D.col_idx.element_size()) + (n + 1) * 4 + 4 * nslab
            + 3 * n * M * 8)
    return {"kernel": f"spmm_kernel<{M}, OP_SPMV(RSUB), double, uint16(slab)> on the "
                      f"{grid}^3 7-pt operator", "algorithmic_bytes": byts,
            "us_per_launch": t * 1e6, "achieved": byts / t / 1e9, "frac": byts / t / 1e9 / peak,
            "timing": "back-to-back launches (each streams the operands from HBM: "
                      f"{byts / 1e6:.0f} MB >> L2), median of 3 rounds of {reps}"}


def spmm_sweep(torch, K, quick: bool):
    """Config 5: blocked SpMM GB/s against the HBM roofline (ASSIGN mode)."""
    from paper_2103_07329_b200 import _lib
    from paper_2103_07329_b200.io import gen_random_sdd
    t0 = time.time()
    A = gen_random_sdd()
    gen_s = time.time() - t0
    peak, _ = peak_hbm()
    out = []
    ms_list = [8] if quick else [1, 2, 4, 8, 16, 32]
    flush_buf = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
    flush_sink = torch.empty((), dtype=torch.float64, device="cuda")
    for vdt in ("f64", "f32"):
        vals = A.values if vdt == "f64" else A.values.astype("float32")
        for idx in ("u32", "u16slab"):
            D = K.DeviceCsr(A.row_ptr, A.col_idx, vals, A.nrows, A.ncols, slab=idx == "u16slab")
            ib = D.col_idx.element_size()
            nslab = 0 if D.slab_base is None else D.slab_base.numel()
            for m, vec in [(m, "f64") for m in ms_list] + [(m, "f32") for m in ms_list
                                                           if vdt == "f32" and idx == "u16slab"]:
                # (fp32 VECTORS -- an extension, loads widened / fp64 accumulation /
                # one rounding at the store -- on the fully compressed format only)
                tdt = torch.float64 if vec == "f64" else torch.float32
                x = torch.rand(A.ncols, m, dtype=tdt, device="cuda")
                y = torch.empty(A.nrows, m, dtype=tdt, device="cuda")
                for _ in range(3):
                    K.csr_spmv(D, None, None, x, y, K.MODE_ASSIGN)
                times = []
                sl0 = _lib.lib().mrs_stream_launches()
                for _ in range(10):
                    torch.sum(flush_buf, dim=0, out=flush_sink)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    K.csr_spmv(D, None, None, x, y, K.MODE_ASSIGN)
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) * 1e-3)
                t = sorted(times)[len(times) // 2]
                vb = 8 if vdt == "f64" else 4
                byts = (A.nnz * (vb + ib) + (A.nrows + 1) * 4 + 4 * nslab
                        + 2 * A.nrows * m * (8 if vec == "f64" else 4))
                out.append({"m": m, "values": vdt, "idx": idx, "vectors": vec, "us": t * 1e6,
                            "GBps": byts / t / 1e9, "frac": byts / t / 1e9 / peak,
                            "kernel": "stream (TMA-fed, csrc/stream.cu)"
                            if _lib.lib().mrs_stream_launches() > sl0 else "lane family (csrc/spmm.cuh)"})
                del x, y
            del D
    return {"n": A.nrows, "nnz": A.nnz, "gen_s": gen_s, "points": out}


def select(name, grid=None):
    global CFG, GRID, M, WORKLOAD, ROLES
    CFG = CONFIGS[name]
    GRID, M = (grid or CFG["grid"]), CFG["m"]
    WORKLOAD, ROLES = CFG["workload"], CFG["roles"]
    if grid and grid != CFG["grid"]:
        WORKLOAD = WORKLOAD + f" [grid {grid}^3]"


def make_matrix():
    from paper_2103_07329_b200 import gen_poisson3d, gen_stencil27_aniso
    if CFG.get("kind") == "s27":
        return gen_stencil27_aniso(GRID, seed=4)
    return gen_poisson3d(GRID, GRID, GRID)[0]


def self_launch(args) -> bool:
    """--gpus N > 1 without a torchrun environment: re-run this script as N
    ranks under torch.distributed.run (one process per GPU, NCCL), forwarding
    every argument; the ranks' rank 0 prints the JSON line.  Returns True when
    the child job ran (its exit status becomes ours)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return False
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    sys.exit(rc)


def main():
    args = parse()
    select(args.config, args.grid)
    self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch "
                         f"{args.gpus} ranks (torchrun) or drop WORLD_SIZE to self-launch")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2103_07329_b200 import BlockVector, gen_poisson3d, kernels as K
    from paper_2103_07329_b200.params import tree
    from paper_2103_07329_b200.solvers import prepare

    A = make_matrix()
    nglob = A.nrows
    Bglob = np.random.default_rng(SEED).uniform(-1.0, 1.0, (nglob, M))
    t0 = time.perf_counter()
    team = None
    partitioned = world > 1 or args.team
    dist_error = None
    if partitioned:
        # row-partitioned solve of the one global system over NCCL (strong scaling)
        try:
            from paper_2103_07329_b200.team import GpuTeam
            team = GpuTeam()
            cs = prepare(tree(ROLES), A, team=team, exec_mode=args.exec)
            lo, hi = cs.row_range
            Bd = torch.from_numpy(np.ascontiguousarray(Bglob[lo:hi])).cuda()
            st = cs.run(Bd, torch.zeros_like(Bd), x_is_zero=True)
            assert st.all_converged, "distributed solve did not converge"
        except Exception as e:        # never leave the driver without a line
            dist_error = f"{type(e).__name__}: {e}"[:300]
            print(f"[bench] distributed path failed ({dist_error}); running replicas",
                  file=sys.stderr)
            partitioned = False
        if dist is not None:
            # every rank takes the same path: replicas as soon as any rank failed
            flag = torch.tensor([0 if partitioned else 1], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            if int(flag.item()) and partitioned:
                partitioned = False
                dist_error = dist_error or "another rank's distributed path failed"
    if not partitioned:
        cs = prepare(tree(ROLES), A, exec_mode=args.exec)
    lo, hi = getattr(cs, "row_range", (0, nglob)) if partitioned else (0, nglob)
    B = np.ascontiguousarray(Bglob[lo:hi])
    n = hi - lo
    plan = cs.plan_factory(M)
    setup_s = time.perf_counter() - t0
    Bd = torch.from_numpy(B).cuda()
    Xd = torch.zeros_like(Bd)
    # L2 flush between timed steps: READ 256 MB (2x the 126 MB L2) so the solve
    # starts cold without inheriting dirty lines to write back
    flush_buf = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
    flush_sink = torch.empty((), dtype=torch.float64, device="cuda")

    def flush_l2():
        torch.sum(flush_buf, dim=0, out=flush_sink)

    clk = ClockSampler(local).__enter__()      # sampled over warm-up, timed loop, soak
    for _ in range(max(args.warmup, 3)):
        st = cs.run(Bd, Xd, x_is_zero=True)
    iters = st.iterations
    assert st.all_converged, "warm-up solve did not converge"

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    step_t = []
    barrier()
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = cs.run(Bd, Xd, x_is_zero=True)
        e1.record()
        e1.synchronize()
        step_t.append(e0.elapsed_time(e1) * 1e-3)
        assert st.iterations == iters
    barrier()
    wall = time.perf_counter() - wall0
    t_dev = sum(step_t)
    if dist is not None:
        tt = torch.tensor([t_dev], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
    # soak ~1 s of the same solves so the clock sampler sees the load (same
    # count on every rank: collectives inside)
    for _ in range(max(1, int(1.0 / max(t_dev / args.steps, 1e-4)))):
        cs.run(Bd, Xd, x_is_zero=True)
    torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    clocks = clk.summary()
    # whole job: one (partitioned) solve per step, or `world` replica solves
    value = (1 if partitioned else world) * M * iters * args.steps / t_dev

    # e2e through the public API with pinned host buffers
    Bh = torch.from_numpy(B).pin_memory()
    Xh = torch.zeros(n, M, dtype=torch.float64).pin_memory()
    Bv = BlockVector(Bh.numpy())
    e2e_t = []
    for k in range(args.warmup + args.steps):
        Xv = BlockVector.zeros(n, M)
        Xv.data = Xh.numpy()
        Xv.flags.zero = True
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st2 = cs.run(Bv, Xv)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            e2e_t.append(dt)
    assert st2.iterations == iters
    e2e_t_max = sum(e2e_t)
    if dist is not None:
        tt = torch.tensor([e2e_t_max], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t_max = float(tt.item())
    e2e_val = (1 if partitioned else world) * M * iters * len(e2e_t) / e2e_t_max
    err = float(np.abs(Xh.numpy() - Xd.cpu().numpy()).max())

    # roofline: the dominant kernel (fine-level SpMM, residual form b - A x, m=8)
    peak, peak_src = peak_hbm()
    A0 = cs.layouts[0].A if partitioned else A          # this rank's block
    D0 = K.DeviceCsr.from_block(A0, slab=True)     # as uploaded by the solver
    Xr = torch.rand(A0.ncols, M, dtype=torch.float64, device="cuda")
    Rd = torch.empty_like(Bd)
    for _ in range(5):
        K.csr_spmv(D0, None, None, Xr, Rd, K.MODE_RSUB, Bd)
    # each launch timed alone after an L2 flush (cold operands, as in the ncu
    # capture that gives `traffic`); median of 50, events on torch's current
    # stream, which is the stream csr_spmv launches on
    reps, kts = 50, []
    for _ in range(reps):
        flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K.csr_spmv(D0, None, None, Xr, Rd, K.MODE_RSUB, Bd)
        e1.record()
        torch.cuda.synchronize()
        kts.append(e0.elapsed_time(e1) * 1e-3)
    kt_cold = sorted(kts)[reps // 2]
    # sustained: back-to-back launches (no per-launch launch latency in the
    # interval) rotating over NSET independent copies of matrix + operands
    # (NSET x ~70 MB >> 126 MB L2), so every launch reads cold operands; the
    # average launch duration = total / launches, events on the launch stream
    nset = max(2, int(math.ceil(3 * 126e6 / max(1.0, (A0.nnz * 10 + 3 * n * M * 8)))) + 1)
    sets = [(K.DeviceCsr.from_block(A0, slab=True), torch.rand_like(Xr), torch.rand_like(Bd),
             torch.empty_like(Rd)) for _ in range(nset)]
    for (Dk, Xk, Bk, Rk) in sets:
        K.csr_spmv(Dk, None, None, Xk, Rk, K.MODE_RSUB, Bk)
    # the 4 x NSET launches are captured into one CUDA graph and replayed: the
    # host's per-call overhead (ctypes, ~10-20 us) never gaps the device
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _r in range(4):
            for (Dk, Xk, Bk, Rk) in sets:
                K.csr_spmv(Dk, None, None, Xk, Rk, K.MODE_RSUB, Bk)
    srounds, skts = 5, []
    for _ in range(srounds):
        flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        skts.append(e0.elapsed_time(e1) * 1e-3 / (4 * nset))
    kt = sorted(skts)[srounds // 2]
    del sets
    nslab = 0 if D0.slab_base is None else D0.slab_base.numel()
    kbytes = (A0.nnz * (A0.values.itemsize + D0.col_idx.element_size()) + (n + 1) * 4 + 4 * nslab
              + (A0.ncols + 2 * n) * M * 8)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"spmm_rsub_{args.config}_g{GRID}_bytes_per_launch")
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": kbytes / kt / 1e9, "peak": peak, "unit": "GB/s",
            "frac": kbytes / kt / 1e9 / peak, "traffic": traffic,
            "kernel": f"spmm_kernel<{M}, OP_SPMV(RSUB), double, uint{8 * D0.col_idx.element_size()}"
                      f"{'(slab)' if nslab else ''}> "
                      f"on the fine-level operator A0 ({args.config})",
            "algorithmic_bytes": kbytes, "us_per_launch": kt * 1e6, "peak_source": peak_src,
            "timing": f"average over back-to-back launches (one captured CUDA graph) rotating "
                      f"{nset} independent cold copies of matrix + operands (CUDA events on the "
                      f"launch stream, median of {srounds} rounds of {4 * nset})",
            "us_per_launch_isolated": kt_cold * 1e6,
            "frac_isolated": kbytes / kt_cold / 1e9 / peak}

    sweep = None
    if not args.no_spmm and rank == 0:
        sweep = spmm_sweep(torch, K, args.quick)
        # the same kernel (fine-level RSUB SpMM of the 7-pt family, m = M, slab
        # indices) where HBM is the binding bound: the 128^3 operator (C3's grid;
        # ~0.5-1 GB per launch >> L2, so back-to-back launches read cold operands)
        if args.config == "c2":
            try:
                roof["at_scale"] = roofline_at_scale(torch, K, peak)
            except Exception as e:       # informational only
                roof["at_scale"] = {"error": f"{type(e).__name__}: {e}"[:200]}

    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        try:
            usable = len(os.sched_getaffinity(0))
        except Exception:
            usable = os.cpu_count() or 1
        res, errs = run_reference_cpu(steps=1, warmup=1, timeout=600, nproc=min(M, usable))
        if res is not None:
            r = res["runs"][0]
            P = res["nproc"]
            cpu = {"value": r[1] / r[0], "unit": UNIT, "cores": P, "kind": "reference",
                   "sample": f"1 full {args.config.upper()} solve ({r[2]} iterations, {r[0]:.2f} s) "
                             f"after a warm-up solve and a {res['setup']:.1f} s reference setup; "
                             f"the m={M} columns over {P} concurrent single-core processes "
                             f"({P} of {os.cpu_count()} host cores), mrsolve {res['backend']} "
                             f"kernels (see --impl reference for the 1-process comparison)"}
        else:
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {errs}"}

    launches = plan.kernel_launches(iters) * args.steps
    try:
        min_bytes = cs.minimal_iteration_bytes(M)
    except Exception as e:           # informational
        print(f"[bench] minimal byte model failed: {e}", file=sys.stderr)
        min_bytes = None
    job_rows = nglob if partitioned else world * n        # rows copied per step, whole job
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
            "scaling": "strong" if partitioned or world == 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: reference 7-pt Poisson generator + default_rng(0).uniform(-1,1) RHS",
            # config: the workload identity only, key-for-key the reference arm's
            "config": {"workload": WORKLOAD, "n": nglob, "m": M, "iterations": iters,
                       "l2": L2_NOTE},
            "details": {"rows_rank0": n,
                       "levels": cs.hierarchy.nlevels if cs.hierarchy is not None else 1,
                       "kernels_per_iteration": plan.kernels_per_iteration,
                       "parallelism": "single GPU" if world == 1 else (
                           f"{world}-GPU row partition + agglomeration, NCCL halo/allreduce"
                           if partitioned else f"{world} replicas (partitioned path failed: "
                                               f"{dist_error})"),
                       "setup_s_excluded": setup_s, "wall_s_timed_region": wall,
                       # two byte models per outer iteration: SURVEY 8(d)'s minimal one
                       # (the algorithm's compulsory traffic) and the plan's own (incl.
                       # its collapsed dense V-cycle tail); whole-solve fraction of the
                       # measured HBM peak from the minimal one
                       "iteration_bytes_minimal": min_bytes,
                       "iteration_bytes_plan": plan.iteration_bytes,
                       "solve_frac_of_hbm_minimal": (min_bytes * iters * args.steps / t_dev / 1e9
                                                     / peak) if min_bytes else None,
                       "final_rel_residual_max": float(st.final_rel_residual.max())},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": job_rows * M * 8,
                    "d2h_bytes_per_step": job_rows * M * 8,
                    "note": "public API run() on pinned host BlockVectors; H2D of B and D2H of "
                            "X inside the timed region", "max_abs_diff_vs_device_run": err},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if sweep is not None:
            line["spmm_sweep"] = sweep
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
