"""The N-rank device path (row partition, halo exchange, split reductions,
agglomeration) executed on ONE GPU through the test-only loopback transport.

Each rank is a distributed plan of this process (team.prepare_distributed,
exactly what GpuTeam ranks build) driven by its own host thread and stream;
``mrs_comm_create_loopback`` replaces NCCL by host barriers + stream events
+ device-to-device copies (csrc/comm.cu), so pack_kernel, the halo landing
offsets (recv_row0 + rdisp), the allreduce -> epilogue split and the
agglomeration all-gather slices all run on the device with NON-EMPTY halos.
No kernel waits on another kernel (B200_PROFILING.md's rule for ranks that
share a GPU).  The product's GpuTeam never selects this transport.

Reference semantics: src/parallel.py:303-355 (halo exchange), src/core.py:
310-404 (partition, segmented blocks).  The distributed dots sum per-rank
partials in rank order (NCCL sums in its own order), so agreement with the
single-GPU solve is by tolerance: iterations equal, X within 1e-10 of the
column's max.
"""

import ctypes as C
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2103_07329_b200 import _lib, gen_poisson3d  # noqa: E402
from paper_2103_07329_b200.io import gen_stencil27_aniso  # noqa: E402
from paper_2103_07329_b200.params import tree  # noqa: E402
from paper_2103_07329_b200.solvers import prepare  # noqa: E402

JAC = {"method": "Jacobi", "weight": "0.8"}
CHEB = {"method": "Chebyshev", "polynomial_order": "2"}
AMG_PCG = {"solver": {"method": "CG", "rel_tolerance": "1e-8"},
           "preconditioner": {"method": "MultiGrid"},
           "pre_smoother": JAC, "post_smoother": JAC}
AMG_BICG_MIXED = {"solver": {"method": "BiCGStab", "rel_tolerance": "1e-8"},
                  "preconditioner": {"method": "MultiGrid", "mg_mixed_precision": "1"},
                  "pre_smoother": CHEB, "post_smoother": CHEB}
AMG_PBICG = {"solver": {"method": "PBiCGStab", "rel_tolerance": "1e-8"},
             "preconditioner": {"method": "MultiGrid"},
             "pre_smoother": JAC, "post_smoother": JAC}


class LoopbackTeam:
    """Duck-typed GpuTeam for one rank of an in-process loopback group."""

    def __init__(self, rank, world, comm, agg_rows_per_rank):
        self.rank, self.world_size, self._comm = rank, world, comm
        self.agg_rows_per_rank = agg_rows_per_rank
        self.force_replicate_from = None

    @property
    def comm(self):
        return self._comm


def loopback_solve(roles, A, B, world, agg_rows):
    L = _lib.lib()
    handles = (C.c_void_p * world)()
    _lib.check(L.mrs_comm_create_loopback(world, handles), "loopback comm")
    teams = [LoopbackTeam(r, world, C.c_void_p(handles[r]), agg_rows) for r in range(world)]
    solvers = [prepare(tree(roles), A, team=t, exec_mode="eager") for t in teams]
    out, errs = [None] * world, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            lo, hi = solvers[r].row_range
            with torch.cuda.stream(torch.cuda.Stream()):
                Bd = torch.from_numpy(np.ascontiguousarray(B[lo:hi])).cuda()
                Xd = torch.zeros_like(Bd)
                st = solvers[r].run(Bd, Xd, x_is_zero=True)
                torch.cuda.current_stream().synchronize()
                out[r] = (st, Xd.cpu().numpy())
        except Exception as e:          # surfaced below
            errs.append((r, e))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    try:
        assert not errs, errs
        assert all(o is not None for o in out), "a rank did not finish"
        X = np.concatenate([o[1] for o in out])
        return [o[0] for o in out], X, solvers
    finally:
        del solvers
        import gc
        gc.collect()
        for r in range(world):
            L.mrs_comm_destroy(C.c_void_p(handles[r]))


def single_solve(roles, A, B):
    Bd = torch.from_numpy(B).cuda()
    Xd = torch.zeros_like(Bd)
    st = prepare(tree(roles), A).run(Bd, Xd, x_is_zero=True)
    return st, Xd.cpu().numpy()


CASES = {
    # name: (matrix, m, roles, agg_rows_per_rank)
    "c2_shrunk": (lambda: gen_poisson3d(24, 24, 24)[0], 8, AMG_PCG, 1500),
    "c3_mixed_shrunk": (lambda: gen_poisson3d(20, 20, 20)[0], 4, AMG_BICG_MIXED, 1000),
    "s27": (lambda: gen_stencil27_aniso(16, seed=4), 8, AMG_PCG, 500),
    "pbicgstab": (lambda: gen_poisson3d(16, 16, 16)[0], 2, AMG_PBICG, 500),
}


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("case", list(CASES))
def test_loopback_ranks_match_single_gpu(case, world):
    mk, m, roles, agg = CASES[case]
    A = mk()
    B = np.random.default_rng(world + 17).uniform(-1.0, 1.0, (A.nrows, m))
    st1, X1 = single_solve(roles, A, B)
    sts, X, solvers = loopback_solve(roles, A, B, world, agg)
    # the halo exchanges and the agglomeration really are non-trivial
    lays = solvers[0].layouts
    assert sum(hp.nrecv for hp in lays[0].halos.values()) > 0
    assert any(l.replicated and l.slice[1] > 0 for l in lays), "no agglomerated level"
    for st in sts:                       # every rank took the same decisions
        assert st.iterations == sts[0].iterations
        np.testing.assert_array_equal(st.final_rel_residual, sts[0].final_rel_residual)
    assert sts[0].iterations == st1.iterations, (sts[0].iterations, st1.iterations)
    assert sts[0].all_converged
    err = np.abs(X - X1).max(axis=0) / np.abs(X1).max(axis=0)
    assert err.max() <= 1e-10, err
    np.testing.assert_allclose(sts[0].final_rel_residual, st1.final_rel_residual, rtol=1e-4)
