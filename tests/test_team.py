"""Multi-GPU host logic on a CPU gloo world of 2 (no GPU needed).

The partition / local-block / halo-plan construction of team.py is exactly
what the device path uploads.  Here each rank exchanges halos with
torch.distributed (gloo) following the plans and runs the oracle SpMM on its
local blocks; the result must equal the rows of the global product BITWISE
(the local blocks keep each row's global entry order).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2103_07329_b200.amg import setup
from paper_2103_07329_b200.io import gen_poisson3d, gen_stencil27_aniso
from paper_2103_07329_b200.team import equal_slices, plan_levels


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def exchange(x_local, nloc, plan, rank, world):
    """Fill the halo segment of x_ext following a HaloPlan (gloo p2p)."""
    m = x_local.shape[1]
    x_ext = np.zeros((nloc + plan.nrecv, m))
    x_ext[:nloc] = x_local
    reqs, off = [], 0
    sends = []
    for p in range(world):
        c = int(plan.send_counts[p])
        if c:
            buf = torch.from_numpy(np.ascontiguousarray(x_local[plan.send_idx[off:off + c]]))
            sends.append(buf)
            reqs.append(dist.isend(buf, p))
        off += c
    recv_bufs, roff = [], nloc
    for p in range(world):
        c = int(plan.recv_counts[p])
        if c:
            buf = torch.empty((c, m), dtype=torch.float64)
            recv_bufs.append((roff, buf))
            reqs.append(dist.irecv(buf, p))
        roff += c
    for r in reqs:
        r.wait()
    for roff, buf in recv_bufs:
        x_ext[roff:roff + buf.shape[0]] = buf.numpy()
    return x_ext


def spmv(blk, x, mode=0, y=None):
    out = np.zeros((blk.nrows, x.shape[1])) if y is None else y
    O.csr_spmv(blk.row_ptr, blk.col_idx, blk.values, np.ascontiguousarray(x), out, mode)
    return out


def worker(rank, world, port, problem, force, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = gen_poisson3d(12, 10, 9)[0] if problem == "p7" else gen_stencil27_aniso(9, seed=4)
        h = setup(A, mixed_precision=True)
        levels = [(lv.A, lv.P, lv.R) for lv in h.levels]
        lays = plan_levels(levels, rank, world, agg_rows_per_rank=64, force_replicate_from=force)
        rng = np.random.default_rng(7)
        m = 3
        checked = 0
        for l, lay in enumerate(lays):
            A_l, P_l, R_l = levels[l]
            n_l = A_l.nrows
            x = rng.standard_normal((n_l, m))
            if lay.replicated:
                continue
            lo, hi = lay.rows
            nloc = hi - lo
            # A_l x
            xe = exchange(x[lo:hi], nloc, lay.halos[0], rank, world)
            assert np.array_equal(spmv(lay.A, xe), spmv(A_l, x)[lo:hi]), f"A level {l}"
            checked += 1
            if P_l is None:
                continue
            # R_l r (partitioned or agglomerated coarse rows)
            re = exchange(x[lo:hi], nloc, lay.halos[1], rank, world)
            rc_local = spmv(lay.R, re)
            rc_full = spmv(R_l, x)
            if lays[l + 1].replicated:
                sl, q = equal_slices(R_l.nrows, world)
                a, b = sl[rank]
                assert np.array_equal(rc_local, rc_full[a:b]), f"R slice level {l}"
                pad = np.zeros((q, m))
                pad[:b - a] = rc_local
                gathered = [torch.empty((q, m), dtype=torch.float64) for _ in range(world)]
                dist.all_gather(gathered, torch.from_numpy(pad))
                full = torch.cat(gathered).numpy()[:R_l.nrows]
                assert np.array_equal(full, rc_full), f"agglomerated R level {l}"
                assert lays[l + 1].slice == (a, q)
                xc = rng.standard_normal((P_l.ncols, m))
                y0 = rng.standard_normal((n_l, m))
                y = y0[lo:hi].copy()
                spmv(lay.P, xc, mode=1, y=y)
                assert np.array_equal(y, spmv(P_l, xc, 1, y0.copy())[lo:hi]), f"P repl {l}"
            else:
                clo, chi = lays[l + 1].rows
                assert np.array_equal(rc_local, rc_full[clo:chi]), f"R level {l}"
                xc = rng.standard_normal((P_l.ncols, m))
                xce = exchange(xc[clo:chi], chi - clo, lay.halos[2], rank, world)
                y0 = rng.standard_normal((n_l, m))
                y = y0[lo:hi].copy()
                spmv(lay.P, xce, mode=1, y=y)
                assert np.array_equal(y, spmv(P_l, xc, 1, y0.copy())[lo:hi]), f"P level {l}"
            checked += 1
        ret[rank] = checked
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("problem,force", [("p7", None), ("p7", 1), ("p27", 2)])
def test_distributed_products_bitwise_gloo_world2(problem, force):
    world = 2
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    mp.spawn(worker, args=(world, _free_port(), problem, force, ret), nprocs=world, join=True)
    assert all(ret[r] >= 1 for r in range(world)), dict(ret)


def test_plan_levels_single_rank_has_no_halos():
    A = gen_poisson3d(8, 8, 8)[0]
    h = setup(A)
    lays = plan_levels([(lv.A, lv.P, lv.R) for lv in h.levels], 0, 1, agg_rows_per_rank=1)
    assert not lays[0].replicated and lays[-1].replicated
    for lay in lays:
        for hp in lay.halos.values():
            assert hp.nsend == 0 and hp.nrecv == 0


def test_local_blocks_use_compressed_indices():
    """Rank-local blocks of a partitioned 27-pt level index < 65536 columns:
    stored as u16 (the reference's index compression of segmented blocks)."""
    A = gen_stencil27_aniso(48, seed=4)          # n = 110592 > 65536: global u32
    assert A.col_idx.dtype == np.uint32
    lays = plan_levels([(A, None, None)], 0, 4)
    assert lays[0].A.col_idx.dtype == np.uint16
    assert lays[0].A.ncols < 65536


def test_slab_compress_roundtrip_and_bandwidth_limit():
    from paper_2103_07329_b200.core import slab_compress
    from paper_2103_07329_b200.io import gen_random_sdd
    A = gen_random_sdd(n=200_000, band=4096, seed=5)
    assert A.col_idx.dtype == np.uint32
    col16, base, shift = slab_compress(A.row_ptr, A.col_idx)
    assert col16.dtype == np.uint16 and (1 << shift) >= 64
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    np.testing.assert_array_equal(base[rows >> shift].astype(np.int64) + col16,
                                  A.col_idx.astype(np.int64))
    # a full-width random matrix cannot be slab-compressed
    rng = np.random.default_rng(0)
    from mrs_testutil import random_csr
    R = random_csr(70001, 70001, 8.0, rng)
    assert slab_compress(R.row_ptr, R.col_idx.astype(np.uint32)) is None


def _setup_worker(rank, world, port, ret):
    """prepare() on a gloo world: rank 0 sets up, every rank receives only its
    own layouts; they equal what the rank would derive from the global setup."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_07329_b200 import amg as amg_mod
        from paper_2103_07329_b200.params import tree
        from paper_2103_07329_b200.solvers import prepare
        from paper_2103_07329_b200.team import GpuTeam
        calls = []
        real = amg_mod.setup

        def counting_setup(*a, **k):
            calls.append(1)
            return real(*a, **k)
        import paper_2103_07329_b200.solvers as S
        S.amg_setup = counting_setup
        A = gen_poisson3d(20, 18, 16)[0]
        roles = {"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"},
                 "pre_smoother": {"method": "Jacobi", "weight": "0.8"},
                 "post_smoother": {"method": "Jacobi", "weight": "0.8"}}
        team = GpuTeam(agg_rows_per_rank=800)
        cs = prepare(tree(roles), A, team=team)
        h = real(A)
        want = plan_levels([(lv.A, lv.P, lv.R) for lv in h.levels], rank, world, 800)
        ok = len(want) == len(cs.layouts) == cs.nlevels
        for a, b in zip(want, cs.layouts):
            ok &= a.rows == b.rows and a.replicated == b.replicated and a.slice == b.slice
            ok &= a.interior == b.interior
            for tag in ("A", "P", "R"):
                x, y = getattr(a, tag), getattr(b, tag)
                ok &= (x is None) == (y is None)
                if x is not None:
                    ok &= np.array_equal(x.row_ptr, y.row_ptr) and np.array_equal(
                        x.col_idx, y.col_idx) and np.array_equal(x.values, y.values)
            for w, hp in a.halos.items():
                ok &= np.array_equal(hp.send_idx, b.halos[w].send_idx)
                ok &= np.array_equal(hp.recv_counts, b.halos[w].recv_counts)
        # a configuration error on rank 0 is raised on every rank
        from paper_2103_07329_b200.errors import ConfigurationError
        bad = {"solver": {"method": "Direct"}}
        raised = False
        try:
            prepare(tree(bad), A, team=team)
        except ConfigurationError:
            raised = True
        ret[rank] = (bool(ok), len(calls), cs.hierarchy is not None, raised)
    finally:
        dist.destroy_process_group()


def test_one_setup_for_all_ranks_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    mp.spawn(_setup_worker, args=(world, _free_port(), ret), nprocs=world, join=True)
    assert ret[0] == (True, 1, True, True), ret[0]       # rank 0: the one setup
    assert ret[1] == (True, 0, False, True), ret[1]      # rank 1: no setup, own blocks only
