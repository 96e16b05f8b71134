"""Multi-GPU team: one process per GPU, row-partitioned hierarchy, NCCL.

Replaces the reference's emulated worker team (src/parallel.py: WorkerTeam,
ExchangePlan / halo_exchange, staged_sum) with real ranks:

* every level is row-partitioned with the reference's rule (core.py:310-344,
  :func:`make_partition`) until it has fewer than ``agg_rows_per_rank`` rows
  per rank; from there on the hierarchy is **agglomerated** -- replicated on
  every rank, fed by an all-gather of the restricted vector;
* a rank's local block keeps each row's global entry order and renumbers its
  columns as [own rows | halo rows ordered by (owner, global id)]: the SpMM
  result of every row is bitwise the single-GPU one, and local column indices
  shrink to 16 bits wherever the block allows (the reference's index
  compression of segmented blocks, core.py:257-270, 364-404);
* halo plans (:class:`HaloPlan`) play the reference's ExchangePlan
  (parallel.py:259-300): import lists are the sorted unique referenced peer
  rows; on the device a pack kernel + grouped ncclSend/ncclRecv fills the halo
  segment before every SpMM whose operand has one;
* dots: local partials -> ncclAllReduce -> the device epilogue (identical
  scalars on every rank).

The host logic here is pure numpy so it is testable on CPU (tests/test_team.py
runs it on a gloo world of 2 and checks distributed SpMMs bitwise against
global ones).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import CsrBlock, choose_width, make_partition
from .errors import ConfigurationError, InvalidArgumentError

__all__ = ["GpuTeam", "HaloPlan", "LevelLayout", "localize", "plan_levels", "equal_slices",
           "prepare_distributed"]


# ---------------------------------------------------------------------------
# partitions and local blocks (host, numpy)
# ---------------------------------------------------------------------------

def equal_slices(n: int, nparts: int):
    """Agglomeration slices: q = ceil(n/nparts) rows each (last one shorter),
    so the all-gathered buffer of nparts*q rows holds the vector in order."""
    q = -(-n // nparts)
    return [(min(r * q, n), min((r + 1) * q, n)) for r in range(nparts)], q


@dataclass
class HaloPlan:
    """Exchange of one gathered operand for one rank."""
    send_idx: np.ndarray                 # int32 local rows, grouped by destination rank
    send_counts: np.ndarray              # int32 [world]
    recv_counts: np.ndarray              # int32 [world]

    @property
    def nrecv(self) -> int:
        return int(self.recv_counts.sum())

    @property
    def nsend(self) -> int:
        return int(self.send_counts.sum())


def _halo_ids(blk: CsrBlock, rows: tuple, cols: tuple) -> np.ndarray:
    lo, hi = rows
    c = blk.col_idx[blk.row_ptr[lo]:blk.row_ptr[hi]].astype(np.int64)
    return np.unique(c[(c < cols[0]) | (c >= cols[1])])


def localize(blk: CsrBlock, rows: tuple, cols: tuple, col_ranges: list | None):
    """Rows [rows) of `blk` with columns renumbered: own column range `cols`
    first, then the halo (sorted global ids).  ``col_ranges`` = every rank's
    column range (None: columns replicated -- no halo).
    Returns (local CsrBlock, halo global ids, recv_counts per rank)."""
    lo, hi = rows
    k0, k1 = int(blk.row_ptr[lo]), int(blk.row_ptr[hi])
    rp = (blk.row_ptr[lo:hi + 1] - k0).astype(np.int64)
    c = blk.col_idx[k0:k1].astype(np.int64)
    v = blk.values[k0:k1]
    if col_ranges is None:
        ncols = blk.ncols
        new = c
        halo = np.zeros(0, dtype=np.int64)
        recv = None
    else:
        own = (c >= cols[0]) & (c < cols[1])
        halo = np.unique(c[~own])
        nloc = cols[1] - cols[0]
        new = np.where(own, c - cols[0], nloc + np.searchsorted(halo, c))
        ncols = nloc + len(halo)
        recv = np.array([np.count_nonzero((halo >= a) & (halo < b)) for a, b in col_ranges],
                        dtype=np.int32)
    width = choose_width(max(ncols, 1))
    local = CsrBlock(hi - lo, ncols, rp, new.astype(width.dtype), v, validate=False)
    return local, halo, recv


def interior_range(local: CsrBlock, nown: int) -> tuple:
    """Longest run [ilo, ihi) of rows of a localized block that read no halo
    column (local column >= nown).  Their product can run while the halo
    exchange is in flight; the other rows run after it (csrc/solver.cu
    spmm_overlapped).  For a z-slab partition of a stencil these are all rows
    but the first and last planes."""
    n = local.nrows
    if n == 0:
        return (0, 0)
    rp = np.asarray(local.row_ptr, dtype=np.int64)
    halo_entry = np.asarray(local.col_idx).astype(np.int64) >= nown
    cum = np.concatenate([[0], np.cumsum(halo_entry, dtype=np.int64)])
    boundary = (cum[rp[1:]] - cum[rp[:-1]]) > 0
    if not boundary.any():
        return (0, n)
    # runs of interior rows between boundary rows
    idx = np.flatnonzero(boundary)
    starts = np.concatenate([[0], idx + 1])
    ends = np.concatenate([idx, [n]])
    k = int(np.argmax(ends - starts))
    return (int(starts[k]), int(ends[k]))


def halo_plan(blk: CsrBlock, row_ranges: list, col_ranges: list, rank: int) -> HaloPlan:
    """My exchange for operand products of `blk`: rows each peer imports from
    me (in its halo order) and my receive counts."""
    world = len(row_ranges)
    my_lo, my_hi = col_ranges[rank]
    send, scount = [], np.zeros(world, dtype=np.int32)
    for p in range(world):
        if p == rank:
            continue
        h = _halo_ids(blk, row_ranges[p], col_ranges[p])
        mine = h[(h >= my_lo) & (h < my_hi)] - my_lo
        send.append(mine.astype(np.int32))
        scount[p] = len(mine)
    h = _halo_ids(blk, row_ranges[rank], col_ranges[rank])
    recv = np.array([np.count_nonzero((h >= a) & (h < b)) for a, b in col_ranges], dtype=np.int32)
    sidx = np.concatenate(send) if send else np.zeros(0, dtype=np.int32)
    return HaloPlan(sidx.astype(np.int32), scount, recv)


@dataclass
class LevelLayout:
    """One rank's view of one level."""
    rows: tuple                    # owned rows (replicated: all)
    replicated: bool
    A: CsrBlock = None
    P: CsrBlock | None = None
    R: CsrBlock | None = None
    halos: dict = field(default_factory=dict)      # 0: A, 1: R, 2: P -> HaloPlan
    interior: dict = field(default_factory=dict)   # 0/1/2 -> (ilo, ihi) rows without halo reads
    slice: tuple = (0, 0)          # agglomeration: (row0, rows) of my restricted slice


def plan_levels(levels: list, rank: int, world: int, agg_rows_per_rank: int = 16384,
                force_replicate_from: int | None = None) -> list:
    """Row partition + local blocks + halo plans of every level for `rank`.

    ``levels``: [(A, P, R)] global blocks (P, R None on the coarsest level).
    Level l is partitioned while n_l / world >= agg_rows_per_rank (and the
    level above is partitioned); ``force_replicate_from`` (tests) replicates
    from that level on regardless.
    """
    n = [lv[0].nrows for lv in levels]
    nl = len(levels)
    repl = []
    for l in range(nl):
        r = (l > 0 and repl[l - 1]) or (l == nl - 1 and nl > 1) or n[l] < world or \
            (l > 0 and n[l] / world < agg_rows_per_rank)
        if force_replicate_from is not None and l >= force_replicate_from:
            r = True
        if l == 0:
            r = False
        repl.append(r)
    ranges = [make_partition(n[l], world, allow_empty=True).ranges if not repl[l]
              else [(0, n[l])] * world for l in range(nl)]
    out = []
    for l, (A, P, R) in enumerate(levels):
        if repl[l]:
            out.append(LevelLayout((0, n[l]), True, A, P, R))
            continue
        rr = ranges[l]
        lay = LevelLayout(rr[rank], False)
        lay.A, _, _ = localize(A, rr[rank], rr[rank], rr)
        lay.halos[0] = halo_plan(A, rr, rr, rank)
        nown = rr[rank][1] - rr[rank][0]
        lay.interior[0] = interior_range(lay.A, nown)
        if P is not None:
            if repl[l + 1]:
                # agglomeration: R restricts my slice of the (replicated) coarse
                # rows; P reads the whole replicated coarse vector
                sl, q = equal_slices(n[l + 1], world)
                lay.R, _, _ = localize(R, sl[rank], rr[rank], rr)
                lay.halos[1] = halo_plan(R, sl, rr, rank)
                lay.interior[1] = interior_range(lay.R, nown)
                lay.P, _, _ = localize(P, rr[rank], (0, n[l + 1]), None)
                out_slice = (sl[rank][0], q)
            else:
                rc = ranges[l + 1]
                lay.R, _, _ = localize(R, rc[rank], rr[rank], rr)
                lay.halos[1] = halo_plan(R, rc, rr, rank)
                lay.P, _, _ = localize(P, rr[rank], rc[rank], rc)
                lay.halos[2] = halo_plan(P, rr, rc, rank)
                lay.interior[1] = interior_range(lay.R, nown)
                lay.interior[2] = interior_range(lay.P, rc[rank][1] - rc[rank][0])
                out_slice = None
            lay._next_slice = out_slice
        out.append(lay)
    # the first replicated level records the slice it is gathered from
    for l in range(1, nl):
        if out[l].replicated and not out[l - 1].replicated:
            row0, q = out[l - 1]._next_slice
            out[l].slice = (row0, q)
    return out


# ---------------------------------------------------------------------------
# the team
# ---------------------------------------------------------------------------

class GpuTeam:
    """One rank per GPU over torch.distributed; owns an NCCL communicator for
    the solve plans.  ``world_size == 1`` is valid (single GPU through the
    distributed code path -- used by tests)."""

    def __init__(self, agg_rows_per_rank: int = 16384, force_replicate_from: int | None = None):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world_size = dist.get_rank(), dist.get_world_size()
        else:
            self.rank, self.world_size = 0, 1
        self.agg_rows_per_rank = agg_rows_per_rank
        self.force_replicate_from = force_replicate_from
        self._comm = None

    @property
    def comm(self):
        if self._comm is None:
            import torch.distributed as dist
            L = _lib.lib()
            buf = (C.c_char * 128)()
            if self.rank == 0:
                _lib.check(L.mrs_comm_unique_id(buf), "nccl unique id")
            uid = [bytes(buf)]
            if self.world_size > 1:
                dist.broadcast_object_list(uid, src=0)
            h = C.c_void_p()
            _lib.check(L.mrs_comm_create(uid[0], self.rank, self.world_size, C.byref(h)),
                       "nccl communicator")
            self._comm = h
        return self._comm

    def row_range(self, n: int) -> tuple:
        return make_partition(n, self.world_size, allow_empty=True).ranges[self.rank]

    def close(self):
        if self._comm is not None:
            _lib.lib().mrs_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _torch_dist():
    import torch.distributed as dist
    return dist if (dist.is_available() and dist.is_initialized()) else None


def _check_team_config(desc):
    if _lib.PC_SGS == desc.precond or _lib.SMOOTH_SGS in (
            (desc.pre.kind, desc.post.kind) if desc.precond == _lib.PC_MG else ()):
        # the reference's hybrid sweep couples leaves through the pre-sweep
        # iterate; the device sweep implements the one-leaf order only
        raise ConfigurationError("Gauss-Seidel smoothing is single-GPU only on the device path")
    if desc.method == _lib.METHOD_DIRECT:
        raise ConfigurationError("the Direct solver (dense inverse) is single-GPU only")


def _rank_payload(cfg, glob, rank, team):
    """Everything rank `rank` uploads: plan descriptor, its layouts (local
    blocks + halo plans + interior ranges), per-level Chebyshev bounds, the
    coarse operators, the method name."""
    desc, levels, inv, h, name, Ab = cfg
    lays = plan_levels(glob, rank, team.world_size, team.agg_rows_per_rank,
                       team.force_replicate_from)
    return {"desc": bytes(desc), "lays": lays, "bounds": [lv[3] for lv in levels],
            "inv": inv, "name": name, "nlevels": len(levels)}


def _scatter_setup(config, A, team, hierarchy, exec_mode, eig_bounds, dist):
    """One setup for the whole team: rank 0 builds the hierarchy, the coarse
    operators and every rank's local blocks, and sends each rank ONLY its own
    (torch.distributed point-to-point object messages, one rank at a time, so
    rank 0 never holds more than one foreign payload).  Other ranks keep host
    memory proportional to their rows.  A setup error on rank 0 is re-raised
    on every rank."""
    from .solvers import _configure
    if team.rank == 0:
        payload, err = None, None
        try:
            cfg = _configure(config, A, hierarchy, exec_mode, eig_bounds)
            _check_team_config(cfg[0])
            glob = [(lv[0], lv[1], lv[2]) for lv in cfg[1]]
        except Exception as e:          # sent to the other ranks, raised everywhere
            err = e
        for r in range(1, team.world_size):
            msg = [err if err is not None else _rank_payload(cfg, glob, r, team)]
            dist.send_object_list(msg, dst=r)
        if err is not None:
            raise err
        payload = _rank_payload(cfg, glob, 0, team)
        return payload, cfg[3]
    msg = [None]
    dist.recv_object_list(msg, src=0)
    if isinstance(msg[0], Exception):
        raise msg[0]
    return msg[0], None


def prepare_distributed(config, A, team: GpuTeam, *, hierarchy=None, exec_mode: str = "graph",
                        eig_bounds=None):
    """``prepare`` on a team.  With a torch.distributed world the setup runs
    ONCE, on rank 0, which sends every rank its own local blocks
    (:func:`_scatter_setup`); without one (a 1-rank team, the test-only
    loopback ranks) each rank derives its blocks from the same deterministic
    global setup.  ``run(B, X)`` takes THIS rank's rows of B and X
    (``team.row_range(n)``)."""
    from .solvers import ConfiguredSolver, DevicePlan, _configure, _vector_args
    from .errors import ShapeMismatchError
    dist = _torch_dist()
    if dist is not None and team.world_size > 1:
        payload, h = _scatter_setup(config, A, team, hierarchy, exec_mode, eig_bounds, dist)
        desc = _lib.mrs_plan_desc.from_buffer_copy(payload["desc"])
    else:
        cfg = _configure(config, A, hierarchy, exec_mode, eig_bounds)
        _check_team_config(cfg[0])
        glob = [(lv[0], lv[1], lv[2]) for lv in cfg[1]]
        payload = _rank_payload(cfg, glob, team.rank, team)
        desc, h = cfg[0], cfg[3]
    lays, inv, name = payload["lays"], payload["inv"], payload["name"]
    if exec_mode == "graph":
        # NCCL p2p/collectives are captured into one ordinary graph per
        # 4 iterations (host checks convergence between launches) rather than
        # into a conditional-node body
        desc.exec = 2
    local_levels = [(lay.A, lay.P, lay.R, payload["bounds"][l]) for l, lay in enumerate(lays)]
    lo, hi = lays[0].rows
    desc.nrows = hi - lo
    plans: dict = {}

    def plan_for(m: int) -> DevicePlan:
        if m not in plans:
            d = _lib.mrs_plan_desc.from_buffer_copy(desc)
            d.m = m
            plans[m] = DevicePlan(d, local_levels, inv, name, dist=(team, lays))
        return plans[m]

    def run(B, X, x_is_zero=None):
        shape, bp, xp, x_zero, host, stream, keep = _vector_args(B, X)
        if x_is_zero is not None:
            x_zero = bool(x_is_zero)
        if shape[0] != hi - lo:
            raise ShapeMismatchError(f"rank {team.rank} owns rows [{lo}, {hi}); got {shape[0]}")
        st = plan_for(shape[1]).solve(bp, xp, x_zero, host, stream)
        if host:
            X.flags.zero = False
            X.flags.initialized = True
        return st

    cs = ConfiguredSolver(name, run, h, plan_for, desc,
                          [(lay.A, lay.P, lay.R) for lay in lays])
    cs.layouts = lays
    cs.row_range = (lo, hi)
    cs.nlevels = payload["nlevels"]
    return cs
