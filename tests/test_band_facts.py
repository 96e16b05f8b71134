"""Host logic behind the single-RHS stream kernel (kernels.band_facts): the
structure facts a DeviceCsr passes to the C ABI (mrs_csr.band / blk_max)."""

import numpy as np

from paper_2103_07329_b200.kernels import band_facts


def test_band_facts_tridiagonal_and_blocks():
    n = 1000
    rows = np.repeat(np.arange(n), 3)
    cols = np.clip(rows + np.tile([-1, 0, 1], n), 0, n - 1)
    rp = np.arange(0, 3 * n + 1, 3)
    band, blk = band_facts(rp, cols.astype(np.uint32))
    assert band == 1
    assert blk == 3 * 256                      # a full aligned block of 256 rows


def test_band_facts_far_entry_ragged_rows_and_empty():
    rp = np.array([0, 2, 2, 5, 6])             # row 1 is empty
    ci = np.array([0, 3, 0, 2, 3, 0], dtype=np.uint32)
    band, blk = band_facts(rp, ci)
    assert band == 3                           # (row 0, col 3) and (row 3, col 0)
    assert blk == 6
    assert band_facts(np.array([0]), np.array([], dtype=np.uint32)) == (-1, 0)
    assert band_facts(np.array([0, 0, 0]), np.array([], dtype=np.uint32)) == (-1, 0)


def test_band_facts_matches_bruteforce(rng):
    n = 5000
    k = rng.poisson(6.0, n)
    rp = np.concatenate(([0], np.cumsum(k)))
    rows = np.repeat(np.arange(n), k)
    ci = np.clip(rows + rng.integers(-700, 701, rows.size), 0, n - 1).astype(np.uint32)
    band, blk = band_facts(rp, ci)
    assert band == int(np.abs(ci.astype(np.int64) - rows).max())
    assert blk == max(int(rp[min(n, r + 256)] - rp[r]) for r in range(0, n, 256))
