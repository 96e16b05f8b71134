"""Oracle restatement of the reference AMG setup (upstream of the hot path).

TEST INFRASTRUCTURE ONLY -- the checker for the product's native setup
(paper_2103_07329_b200/csrc/amg_setup.cpp).  Follows
/root/reference/pkg/src/mrsolve/amg.py:

* strength_graph   amg.py:55-78   classical negative-coupling rule
* coarsen          amg.py:89-124  index-ordered greedy C/F split (+aggressive)
* interpolate      amg.py:127-182 direct interpolation
* galerkin         amg.py:185-196 R A P with scipy's sparse products
* setup            amg.py:254-308 level loop, stall cut-off, retry once,
                                  mixed-precision tagging (l >= 1 -> float32)

Pinned against tests/golden/hierarchies.npz (reference output).  Uses plain
Python loops: only for the small sizes the tests use.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .oracle import Csr, Hierarchy, Level

U, C, F = 0, 1, 2


def strength(A: sp.csr_matrix, theta: float) -> sp.csr_matrix:
    n = A.shape[0]
    coo = A.tocoo()
    off = coo.row != coo.col
    rows, cols, vals = coo.row[off], coo.col[off], coo.data[off]
    neg = -vals
    rowmax = np.zeros(n)
    np.maximum.at(rowmax, rows, neg)
    keep = (rowmax[rows] > 0) & (neg >= theta * rowmax[rows])
    S = sp.csr_matrix((np.ones(int(keep.sum()), dtype=bool), (rows[keep], cols[keep])),
                      shape=(n, n))
    S.sort_indices()
    return S


def split(S: sp.csr_matrix, aggressive: bool, num_paths: int) -> np.ndarray:
    n = S.shape[0]
    ST = S.T.tocsr()
    ST.sort_indices()
    ip, ix = ST.indptr, ST.indices
    state = np.zeros(n, dtype=np.int8)
    for i in range(n):
        if state[i] != U:
            continue
        state[i] = C
        dep = ix[ip[i]:ip[i + 1]]
        state[dep[state[dep] == U]] = F
        if aggressive and len(dep):
            hop = np.concatenate([ix[ip[k]:ip[k + 1]] for k in dep])
            if len(hop):
                cand, cnt = np.unique(hop, return_counts=True)
                state[cand[(cnt >= num_paths) & (state[cand] == U) & (cand != i)]] = F
    return state


class _Degenerate(Exception):
    def __init__(self, rows):
        self.rows = rows


def interp(A: sp.csr_matrix, S: sp.csr_matrix, state: np.ndarray) -> sp.csr_matrix:
    n = A.shape[0]
    cpts = np.flatnonzero(state == C)
    cmap = np.full(n, -1, dtype=np.int64)
    cmap[cpts] = np.arange(len(cpts))
    rows, cols, vals, bad = [], [], [], []
    for i in range(n):
        if state[i] == C:
            rows.append(i); cols.append(cmap[i]); vals.append(1.0)
            continue
        lo, hi = A.indptr[i], A.indptr[i + 1]
        ci, vi = A.indices[lo:hi], A.data[lo:hi]
        dmask = ci == i
        a_ii = vi[dmask].sum()
        off_sum = vi[~dmask].sum()
        strong = set(S.indices[S.indptr[i]:S.indptr[i + 1]].tolist())
        sel = np.array([(c in strong and state[c] == C) for c in ci], dtype=bool)
        if not sel.any():
            bad.append(i)
            continue
        w = -(vi[sel] / a_ii) * (off_sum / vi[sel].sum())
        rows.extend([i] * int(sel.sum())); cols.extend(cmap[ci[sel]].tolist())
        vals.extend(w.tolist())
    if bad:
        raise _Degenerate(bad)
    P = sp.csr_matrix((vals, (rows, cols)), shape=(n, len(cpts)))
    P.sort_indices()
    return P


def _canon(M: sp.csr_matrix) -> sp.csr_matrix:
    M = sp.csr_matrix(M)
    M.sort_indices()
    M.sum_duplicates()
    return M


def setup(A: Csr, theta=0.25, agg_num_levels=0, num_paths=1, coarse_size=500,
          max_levels=25, mixed=False, stall_ratio=0.9) -> Hierarchy:
    As = _canon(sp.csr_matrix((A.values.astype(np.float64), A.col_idx.astype(np.int64),
                               A.row_ptr), shape=(A.nrows, A.ncols)))
    chain, Ps = [As], []
    while chain[-1].shape[0] > coarse_size and len(chain) < max_levels:
        M = chain[-1]
        S = strength(M, theta)
        agg = len(chain) - 1 < agg_num_levels
        st = split(S, agg, num_paths)
        try:
            P = interp(M, S, st)
        except _Degenerate as e:
            st = st.copy()
            st[np.asarray(e.rows, dtype=np.int64)] = C
            P = interp(M, S, st)
        P = _canon(P)
        nc = P.shape[1]
        if nc == 0 or nc > stall_ratio * M.shape[0]:
            break
        R = _canon(P.T.tocsr())
        Ac = _canon((R @ M @ P).tocsr())
        Ps.append(P)
        chain.append(Ac)
    levels = []
    for l, M in enumerate(chain):
        dt = np.float32 if (mixed and l > 0) else np.float64
        lv = Level(Csr.from_scipy(M, dt))
        if l < len(Ps):
            P = Ps[l]
            R = _canon(P.T.tocsr())
            lv.P, lv.R = Csr.from_scipy(P, dt), Csr.from_scipy(R, dt)
        levels.append(lv)
    return Hierarchy(levels)
