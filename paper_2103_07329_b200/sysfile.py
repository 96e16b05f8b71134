"""System files and run configurations on either side of the solve path
(SURVEY.md 8(f) rank 4): the reference's ``XAMGBIN1`` binary system format
and its YAML run configuration, so GPU runs read the same inputs.

Format contract (reference /root/reference/pkg/src/mrsolve/io.py:1-20,
:46-149; pinned by its tests/test_io.py): little-endian; a 41-byte header
``magic[8] = b"XAMGBIN1" | nrows, ncols, nnz, nrhs : u64 | flags : u8``
(bit 0 right-hand side present, bit 1 initial guess present), then
``row_ptr u64[nrows+1] | col_idx u64[nnz] | values f64[nnz]`` and the
optional (nrows, nrhs) row-major f64 blocks.  Every malformation raises
``FormatError`` carrying the byte offset where the reference reports it.

Run configuration (io.py:205-283): top-level keys are the four ParamTree
roles plus ``system`` (exactly one of ``poisson: [nx, ny, nz]`` or
``file: path``) and an optional ``benchmark`` (``m``, ``repetitions``,
``mode``).  Host-side only: no device work happens here.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import BlockVector, CsrBlock
from .errors import ConfigurationError, FormatError, InvalidArgumentError
from .params import ROLES, ParamTree

__all__ = ["MAGIC", "read_system", "write_system", "SystemSpec", "BenchmarkSpec",
           "parse_run_config"]

MAGIC = b"XAMGBIN1"
_HDR = np.dtype([("magic", "S8"), ("nrows", "<u8"), ("ncols", "<u8"), ("nnz", "<u8"),
                 ("nrhs", "<u8"), ("flags", "u1")])
_OFF_NRHS = 32          # byte offsets of header fields named in errors
_OFF_FLAGS = 40
assert _HDR.itemsize == 41


def write_system(path, matrix, rhs=None, guess=None):
    """Write ``matrix`` (+ optional rhs / guess block vectors) to ``path``."""
    vecs = [v for v in (rhs, guess) if v is not None]
    if matrix.nrows == 0:
        raise InvalidArgumentError("an empty (0-row) matrix cannot be written")
    for v in vecs:
        if v.data.shape[0] != matrix.nrows:
            raise InvalidArgumentError(
                f"vector has {v.data.shape[0]} rows, matrix has {matrix.nrows}")
    widths = {v.data.shape[1] for v in vecs}
    if len(widths) > 1:
        raise InvalidArgumentError(f"rhs and guess have different column counts {sorted(widths)}")
    hdr = np.zeros((), dtype=_HDR)
    hdr["magic"], hdr["nrows"], hdr["ncols"] = MAGIC, matrix.nrows, matrix.ncols
    hdr["nnz"] = int(np.asarray(matrix.row_ptr)[-1])
    hdr["nrhs"] = widths.pop() if widths else 0
    hdr["flags"] = (1 if rhs is not None else 0) | (2 if guess is not None else 0)
    parts = [hdr.tobytes(), np.asarray(matrix.row_ptr, dtype="<u8").tobytes(),
             np.asarray(matrix.col_idx, dtype="<u8").tobytes(),
             np.asarray(matrix.values, dtype="<f8").tobytes()]
    parts += [np.ascontiguousarray(v.data, dtype="<f8").tobytes() for v in vecs]
    with open(path, "wb") as fh:
        for p in parts:
            fh.write(p)


class _Cursor:
    """Sequential typed reads from the file image; truncation -> FormatError
    at the section's start offset."""

    def __init__(self, buf: bytes, pos: int):
        self.buf, self.pos = buf, pos

    def take(self, dtype: str, count: int, section: str) -> np.ndarray:
        dt = np.dtype(dtype)
        need = dt.itemsize * count
        have = len(self.buf) - self.pos
        if need > have:
            raise FormatError(f"{section}: {need} bytes needed, only {have} left (truncated)",
                              offset=self.pos)
        out = np.frombuffer(self.buf, dtype=dt, count=count, offset=self.pos)
        self.pos += need
        return out


def read_system(path):
    """Read ``(CsrBlock, rhs BlockVector | None, guess BlockVector | None)``.
    Rows stored unsorted are sorted; the block then passes the full CSR
    validation (duplicates etc. -> FormatError at the header end)."""
    with open(path, "rb") as fh:
        buf = fh.read()
    if len(buf) < _HDR.itemsize:
        raise FormatError("shorter than the 41-byte header", offset=0)
    h = np.frombuffer(buf, dtype=_HDR, count=1)[0]
    if bytes(h["magic"]) != MAGIC:
        raise FormatError(f"magic {bytes(h['magic'])!r} is not {MAGIC!r}", offset=0)
    nrows, ncols, nnz, nrhs = (int(h[k]) for k in ("nrows", "ncols", "nnz", "nrhs"))
    flags = int(h["flags"])
    if flags & 0xFC:
        raise FormatError(f"undefined flag bits set (flags = 0x{flags:02x})", offset=_OFF_FLAGS)
    if flags and nrhs == 0:
        raise FormatError("vector blocks flagged but nrhs = 0", offset=_OFF_NRHS)
    cur = _Cursor(buf, _HDR.itemsize)
    rp_at = cur.pos
    rp = cur.take("<u8", nrows + 1, "row_ptr").astype(np.int64)
    if nrows and rp[-1] != nnz:
        raise FormatError(f"row_ptr ends at {rp[-1]}, header says nnz = {nnz}",
                          offset=rp_at + 8 * nrows)
    dec = np.flatnonzero(rp[1:] < rp[:-1])
    if dec.size:
        raise FormatError(f"row_ptr is not non-decreasing (entry {dec[0] + 1})",
                          offset=rp_at + 8 * (int(dec[0]) + 1))
    ci_at = cur.pos
    ci = cur.take("<u8", nnz, "col_idx")
    bad = np.flatnonzero(ci >= ncols)
    if bad.size:
        raise FormatError(f"column index {int(ci[bad[0]])} out of range (ncols = {ncols})",
                          offset=ci_at + 8 * int(bad[0]))
    vals = cur.take("<f8", nnz, "values")
    block = _ingest(nrows, ncols, rp, ci.astype(np.int64), vals.astype(np.float64))
    blocks = []
    for bit, name in ((1, "rhs"), (2, "guess")):
        if flags & bit:
            d = cur.take("<f8", nrows * nrhs, name).astype(np.float64).reshape(nrows, nrhs)
            blocks.append(BlockVector.from_array(d))
        else:
            blocks.append(None)
    if cur.pos != len(buf):
        raise FormatError(f"{len(buf) - cur.pos} trailing bytes after the last section",
                          offset=cur.pos)
    return block, blocks[0], blocks[1]


def _ingest(nrows, ncols, rp, ci, vals) -> CsrBlock:
    """Sort each row's entries by column (stable), then validate as CsrBlock."""
    order = np.lexsort((ci, np.repeat(np.arange(nrows, dtype=np.int64), np.diff(rp))))
    try:
        return CsrBlock.from_arrays(nrows, ncols, rp, ci[order], vals[order], validate=True)
    except InvalidArgumentError as exc:
        raise FormatError(f"matrix violates the CSR invariants: {exc}",
                          offset=_HDR.itemsize) from exc


# ---------------------------------------------------------------------------
# YAML run configuration
# ---------------------------------------------------------------------------

@dataclass
class SystemSpec:
    """Source of the linear system: ``kind`` "poisson" (dims) or "file" (path)."""
    kind: str
    dims: tuple | None = None
    path: str | None = None


@dataclass
class BenchmarkSpec:
    m_list: list = field(default_factory=lambda: [1])
    repetitions: int = 3
    mode: str = "solve"


def _positive_ints(v) -> bool:
    return all(isinstance(x, int) and not isinstance(x, bool) and x >= 1 for x in v)


def parse_run_config(path):
    """``(ParamTree finalized, SystemSpec, BenchmarkSpec)`` from a YAML file;
    the tree equals the programmatic add_map + set_defaults sequence."""
    import yaml
    with open(path) as fh:
        doc = yaml.safe_load(fh)
    where = str(path)
    if not isinstance(doc, dict):
        raise ConfigurationError(f"{where}: the document must be a mapping")
    allowed = set(ROLES) | {"system", "benchmark"}
    extra = [k for k in doc if k not in allowed]
    if extra:
        raise ConfigurationError(f"{where}: unknown top-level key {extra[0]!r} "
                                 f"(allowed: {sorted(allowed)})")
    tree = ParamTree()
    for role in (r for r in ROLES if r in doc):
        if not isinstance(doc[role], dict):
            raise ConfigurationError(f"{where}: {role}: must be a mapping")
        try:
            tree.add_map(role, doc[role])
        except ConfigurationError as exc:
            raise ConfigurationError(f"{where}: {role}: {exc}") from exc
    try:
        tree.set_defaults()
    except ConfigurationError as exc:
        raise ConfigurationError(f"{where}: {exc}") from exc

    sysd = doc.get("system")
    if sysd is None:
        raise ConfigurationError(f"{where}: the 'system' section is required")
    if not isinstance(sysd, dict) or len(sysd) != 1:
        raise ConfigurationError(f"{where}: system: needs exactly one of 'poisson' / 'file'")
    (src, val), = sysd.items()
    if src == "poisson":
        if not (isinstance(val, (list, tuple)) and len(val) == 3 and _positive_ints(val)):
            raise ConfigurationError(f"{where}: system/poisson: three positive integers expected")
        spec = SystemSpec("poisson", dims=tuple(val))
    elif src == "file":
        spec = SystemSpec("file", path=str(val))
    else:
        raise ConfigurationError(f"{where}: system: unknown source {src!r}")

    bench = BenchmarkSpec()
    bd = doc.get("benchmark")
    if bd is not None:
        if not isinstance(bd, dict):
            raise ConfigurationError(f"{where}: benchmark: must be a mapping")
        for key, val in bd.items():
            if key == "m":
                ms = [val] if isinstance(val, int) else list(val)
                if not _positive_ints(ms):
                    raise ConfigurationError(f"{where}: benchmark/m: positive integers expected")
                bench.m_list = ms
            elif key == "repetitions":
                if not (isinstance(val, int) and not isinstance(val, bool) and val >= 1):
                    raise ConfigurationError(
                        f"{where}: benchmark/repetitions: a positive integer expected")
                bench.repetitions = val
            elif key == "mode":
                bench.mode = str(val)
            else:
                raise ConfigurationError(f"{where}: benchmark/{key}: unknown key")
    return tree, spec, bench
