"""XAMGBIN1 system files and YAML run configurations:
the cases the reference pins in tests/test_io.py:22-226, 233-323 -- byte-exact
round trips, the header layout, and the byte offset of every rejection."""

import struct

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_2103_07329_b200.core import BlockVector, CsrBlock
from paper_2103_07329_b200.errors import ConfigurationError, FormatError, InvalidArgumentError
from paper_2103_07329_b200.io import (MAGIC, gen_poisson3d, parse_run_config, read_system,
                                      write_system)
from paper_2103_07329_b200.params import ParamTree

HDR = 41


def system(rng, n=60, m=2):
    a = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.15)
    np.fill_diagonal(a, rng.standard_normal(n) + 5.0)
    return (CsrBlock.from_dense(a), BlockVector.from_array(rng.standard_normal((n, m))),
            BlockVector.from_array(rng.standard_normal((n, m))))


@pytest.fixture
def rng():
    return np.random.default_rng(77)


def written(tmp_path, rng, n=10, **kw):
    mat, rhs, guess = system(rng, n=n)
    p = tmp_path / "s.bin"
    write_system(p, mat, rhs if kw.get("rhs", True) else None,
                 guess if kw.get("guess", True) else None)
    return p, bytearray(p.read_bytes()), mat


def test_round_trip_is_bit_exact(tmp_path, rng):
    mat, rhs, guess = system(rng)
    p = tmp_path / "a.bin"
    write_system(p, mat, rhs, guess)
    m2, r2, g2 = read_system(p)
    for a, b in ((m2.row_ptr, mat.row_ptr), (m2.col_idx, mat.col_idx), (m2.values, mat.values),
                 (r2.data, rhs.data), (g2.data, guess.data)):
        np.testing.assert_array_equal(a, b)


def test_header_layout(tmp_path):
    mat = CsrBlock.from_dense(np.array([[2.0, -1.0], [-1.0, 2.0]]))
    p = tmp_path / "h.bin"
    write_system(p, mat)
    raw = p.read_bytes()
    assert raw[:8] == MAGIC == b"XAMGBIN1"
    assert struct.unpack_from("<QQQQB", raw, 8) == (2, 2, 4, 0, 0)
    np.testing.assert_array_equal(np.frombuffer(raw, "<u8", 3, offset=HDR), [0, 2, 4])
    assert len(raw) == HDR + 8 * 3 + 8 * 4 + 8 * 4


def test_sixteen_rhs_and_matrix_only(tmp_path, rng):
    mat, _, _ = system(rng, n=20)
    rhs = BlockVector.from_array(rng.standard_normal((20, 16)))
    p = tmp_path / "m16.bin"
    write_system(p, mat, rhs)
    assert struct.unpack_from("<QB", p.read_bytes(), 32) == (16, 1)
    _, r2, g2 = read_system(p)
    assert r2.data.shape == (20, 16) and g2 is None
    write_system(p, mat)
    m2, r2, g2 = read_system(p)
    assert r2 is None and g2 is None
    np.testing.assert_array_equal(m2.to_dense(), mat.to_dense())


@given(seed=st.integers(0, 2 ** 31), n=st.integers(1, 30), m=st.integers(1, 4))
@settings(max_examples=20, deadline=None)
def test_round_trip_property(tmp_path_factory, seed, n, m):
    r = np.random.default_rng(seed)
    a = r.standard_normal((n, n)) * (r.random((n, n)) < 0.3)
    np.fill_diagonal(a, 1.0)
    mat = CsrBlock.from_dense(a)
    rhs = BlockVector.from_array(r.standard_normal((n, m)))
    p = tmp_path_factory.mktemp("rt") / "p.bin"
    write_system(p, mat, rhs)
    m2, r2, _ = read_system(p)
    np.testing.assert_array_equal(m2.to_dense(), mat.to_dense())
    np.testing.assert_array_equal(r2.data, rhs.data)


def test_unsorted_rows_are_sorted_on_read(tmp_path):
    mat = CsrBlock.from_dense(np.array([[4.0, 1.0, 2.0], [0.0, 3.0, 0.0], [5.0, 0.0, 6.0]]))
    p = tmp_path / "u.bin"
    write_system(p, mat)
    raw = bytearray(p.read_bytes())
    ci0 = HDR + 8 * 4
    v0 = ci0 + 8 * mat.nnz
    # reverse row 0's three entries in the file
    cols = list(struct.unpack_from("<3Q", raw, ci0))
    vals = list(struct.unpack_from("<3d", raw, v0))
    struct.pack_into("<3Q", raw, ci0, *cols[::-1])
    struct.pack_into("<3d", raw, v0, *vals[::-1])
    p.write_bytes(raw)
    np.testing.assert_array_equal(read_system(p)[0].to_dense(), mat.to_dense())


def test_write_validation(tmp_path, rng):
    mat, _, _ = system(rng, n=10)
    with pytest.raises(InvalidArgumentError):
        write_system(tmp_path / "x.bin", mat, BlockVector.from_array(np.ones((11, 1))))
    with pytest.raises(InvalidArgumentError):
        write_system(tmp_path / "x.bin", mat, BlockVector.from_array(np.ones((10, 2))),
                     BlockVector.from_array(np.ones((10, 3))))


def corrupt_and_read(p, raw):
    p.write_bytes(bytes(raw))
    with pytest.raises(FormatError) as ei:
        read_system(p)
    return ei.value


def test_rejection_offsets(tmp_path, rng):
    n = 10
    p, raw, mat = written(tmp_path, rng, n=n)
    bad = bytearray(raw); bad[:8] = b"NOTMAGIC"
    assert corrupt_and_read(p, bad).offset == 0
    bad = bytearray(raw); bad[40] |= 0x4
    assert corrupt_and_read(p, bad).offset == 40
    bad = bytearray(raw); struct.pack_into("<Q", bad, HDR + 8 * n, 999999)
    e = corrupt_and_read(p, bad)
    assert e.offset == HDR + 8 * n and "nnz" in str(e)
    bad = bytearray(raw); struct.pack_into("<Q", bad, HDR + 8, 5); struct.pack_into("<Q", bad, HDR + 16, 1)
    assert "non-decreasing" in str(corrupt_and_read(p, bad))
    col0 = HDR + 8 * (n + 1)
    bad = bytearray(raw); struct.pack_into("<Q", bad, col0, n + 5)
    e = corrupt_and_read(p, bad)
    assert e.offset == col0 and "out of range" in str(e)
    assert "truncated" in str(corrupt_and_read(p, raw[: len(raw) // 2]))
    e = corrupt_and_read(p, raw + b"\x00" * 16)
    assert "trailing" in str(e) and e.offset == len(raw)
    assert corrupt_and_read(p, b"XAMG").offset == 0


def test_vector_flag_without_nrhs(tmp_path, rng):
    p, raw, _ = written(tmp_path, rng, n=5, rhs=False, guess=False)
    raw[40] |= 0x1
    assert corrupt_and_read(p, raw).offset == 32


def test_duplicate_entries_fail_csr_validation(tmp_path):
    mat = CsrBlock.from_dense(np.array([[1.0, 2.0], [0.0, 3.0]]))
    p = tmp_path / "d.bin"
    write_system(p, mat)
    raw = bytearray(p.read_bytes())
    struct.pack_into("<Q", raw, HDR + 8 * 3 + 8, 0)      # row 0: columns (0, 0)
    assert corrupt_and_read(p, raw).offset == HDR


def test_generated_system_file_drives_the_solver_api(tmp_path):
    """A Poisson system written with its rhs reads back bitwise: files and
    generators feed prepare() identically."""
    A, b = gen_poisson3d(6, 5, 4)
    p = tmp_path / "poisson.bin"
    write_system(p, A, b)
    A2, b2, g2 = read_system(p)
    assert g2 is None
    np.testing.assert_array_equal(A2.to_dense(), A.to_dense())
    np.testing.assert_array_equal(b2.data, b.data)


# ---- YAML run configuration --------------------------------------------------

def cfg(tmp_path, text):
    p = tmp_path / "run.yml"
    p.write_text(text)
    return p


def test_full_run_config(tmp_path):
    tree, system_, bench = parse_run_config(cfg(tmp_path, """
solver:
  method: PBiCGStab
  rel_tolerance: 1e-9
preconditioner:
  method: MultiGrid
  mg_agg_num_levels: 2
  mg_num_paths: 2
pre_smoother:
  method: Chebyshev
post_smoother:
  method: Chebyshev
system:
  poisson: [32, 32, 32]
benchmark:
  m: [1, 2, 4]
  repetitions: 5
"""))
    assert tree.finalized and tree.role("solver").method == "PBiCGStab"
    assert tree.role("preconditioner").get_int("mg_num_paths") == 2
    assert system_.kind == "poisson" and system_.dims == (32, 32, 32)
    assert bench.m_list == [1, 2, 4] and bench.repetitions == 5 and bench.mode == "solve"


def test_run_config_equals_programmatic_tree(tmp_path):
    tree, _, _ = parse_run_config(cfg(tmp_path, """
solver:
  method: BiCGStab
  merged: 1
preconditioner:
  method: MultiGrid
system:
  poisson: [8, 8, 8]
"""))
    manual = ParamTree()
    manual.add_map("solver", {"method": "BiCGStab", "merged": "1"})
    manual.add_map("preconditioner", {"method": "MultiGrid"})
    manual.set_defaults()
    assert tree == manual


def test_file_system_and_benchmark_defaults(tmp_path):
    _, system_, bench = parse_run_config(cfg(tmp_path, "solver:\n  method: CG\nsystem:\n"
                                                       "  file: /data/system.bin\n"))
    assert system_.kind == "file" and system_.path == "/data/system.bin"
    assert (bench.m_list, bench.repetitions, bench.mode) == ([1], 3, "solve")


@pytest.mark.parametrize("text,fragment", [
    ("solver:\n  method: CG\n", "system"),
    ("system:\n  poisson: [2, 2, 2]\n", "solver"),
    ("solver:\n  method: CG\nsystem:\n  poisson: [2, 2]\n", "poisson"),
    ("solver:\n  method: CG\nsystem:\n  poisson: [2, 2, 0]\n", "poisson"),
    ("solver:\n  method: CG\nsystem:\n  lattice: [2, 2, 2]\n", "system"),
    ("solver:\n  method: CG\nsystem:\n  poisson: [2, 2, 2]\nmatrix: x\n", "matrix"),
    ("solver:\n  method: Newton\nsystem:\n  poisson: [2, 2, 2]\n", "Newton"),
    ("solver:\n  method: CG\n  merged: 1\nsystem:\n  poisson: [2, 2, 2]\n", "merged"),
    ("solver:\n  method: CG\nsystem:\n  poisson: [2, 2, 2]\nbenchmark:\n  warmup: 2\n",
     "warmup"),
])
def test_run_config_rejections_carry_context(tmp_path, text, fragment):
    with pytest.raises(ConfigurationError, match=fragment):
        parse_run_config(cfg(tmp_path, text))


def test_reads_and_writes_the_reference_file_byte_for_byte(tmp_path):
    """tests/golden/xamgbin1_ref.bin was written by the reference's
    write_system (oracle/gen_golden.py gen_sysfile)."""
    from mrs_testutil import GOLDEN
    import os
    ref = os.path.join(GOLDEN, "xamgbin1_ref.bin")
    A, rhs, guess = read_system(ref)
    A0, _ = gen_poisson3d(3, 2, 2)
    np.testing.assert_array_equal(A.to_dense(), A0.to_dense())
    r = np.random.default_rng(41)
    np.testing.assert_array_equal(rhs.data, r.standard_normal((A0.nrows, 3)))
    np.testing.assert_array_equal(guess.data, r.standard_normal((A0.nrows, 3)))
    out = tmp_path / "ours.bin"
    write_system(out, A, rhs, guess)
    assert out.read_bytes() == open(ref, "rb").read()
