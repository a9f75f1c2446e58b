"""ARVT table files (the reference's format, approxrv/tableio.py:30-223).

Binary layout (all little-endian):

    offset 0   4s   magic  b"ARVT"
           4   u16  version (1)
           6   u8   kind   0 constant | 1 dyadic | 2 ncchi2 | 3 subdyadic (extension)
           7   u8   degree (0 for constant)
           8   ...  kind-specific header fields, then the f64 coefficient block
          -4   u32  CRC-32 of bytes [8, len-4)

    constant   u32 q, u32 construction index (tables.CONSTRUCTIONS), f64[2^q]
    dyadic     u32 n_intervals, f64 decay, f64[(degree+1) (K+1)]
    ncchi2     f64 nu, u32 n_knots, u32 n_intervals, f64 decay,
               f64 lower[n_knots][degree+1][K+1], f64 upper[...]   (lower first)
    subdyadic  u32 n_octaves, u32 sub_bits, f64[(degree+1) K 2^sub_bits]

The text variant starts with ``# ARVT v1 <kind>``, then ``# key = value``
metadata and one coefficient per line (``%.17g``, exact for f64).  Files the
reference writes load here unchanged and vice versa (byte-identical output
for the three reference kinds); the errors are the reference's
(BadMagicError, VersionError, ChecksumError, TruncatedFileError).
"""

from __future__ import annotations

import struct
import zlib
from pathlib import Path

import numpy as np

from .errors import BadMagicError, ChecksumError, ConfigError, TableIOError, TruncatedFileError, VersionError
from .tables import CONSTRUCTIONS, ConstantTable, DyadicPolyTable, NcChi2Table, SubDyadicTable

MAGIC = b"ARVT"
VERSION = 1
KIND_CONSTANT, KIND_DYADIC, KIND_NCCHI2, KIND_SUBDYADIC = 0, 1, 2, 3
_KIND_WORD = {KIND_CONSTANT: "constant", KIND_DYADIC: "dyadic", KIND_NCCHI2: "ncchi2", KIND_SUBDYADIC: "subdyadic"}
_HEAD = struct.Struct("<4sHBB")  # magic, version, kind, degree
_CRC = struct.Struct("<I")
# kind -> header struct following the 8-byte preamble
_FIELDS = {
    KIND_CONSTANT: struct.Struct("<II"),
    KIND_DYADIC: struct.Struct("<Id"),
    KIND_NCCHI2: struct.Struct("<dIId"),
    KIND_SUBDYADIC: struct.Struct("<II"),
}


def _kind_of(table) -> int:
    name = type(table).__name__
    if isinstance(table, SubDyadicTable):
        return KIND_SUBDYADIC
    for kind, cls in ((KIND_CONSTANT, ConstantTable), (KIND_DYADIC, DyadicPolyTable), (KIND_NCCHI2, NcChi2Table)):
        if isinstance(table, cls) or name == cls.__name__:
            return kind
    raise ConfigError(f"cannot serialize object of type {name}")


def _ncchi2_halves(table):
    """(lower, upper) stacks, each (n_knots, degree+1, K+1)."""
    st = np.asarray(table.eval_stacks)  # upper at 0, lower at 1 (tables.py:148-153)
    return st[1], st[0]


def _encode(table) -> tuple[int, int, bytes, np.ndarray]:
    kind = _kind_of(table)
    if kind == KIND_CONSTANT:
        return kind, 0, _FIELDS[kind].pack(table.q, CONSTRUCTIONS.index(table.construction)), table.values
    if kind == KIND_DYADIC:
        return kind, table.degree, _FIELDS[kind].pack(table.n_intervals, table.decay), table.coeffs
    if kind == KIND_NCCHI2:
        lower, upper = _ncchi2_halves(table)
        decay = getattr(table, "decay", None)
        if decay is None:
            decay = table.lower[0].decay if hasattr(table, "lower") else 0.5
        head = _FIELDS[kind].pack(table.nu, table.n_knots, table.n_intervals, decay)
        return kind, table.degree, head, np.concatenate([lower.reshape(-1), upper.reshape(-1)])
    return kind, table.degree, _FIELDS[kind].pack(table.n_octaves, table.sub_bits), table.coeffs


def export_table(table, path, format: str = "binary") -> None:
    """Write ``table`` to ``path`` as a binary (default) or text ARVT file."""
    if format not in ("binary", "text"):
        raise ConfigError(f"unknown table format {format!r}")
    kind, degree, head, block = _encode(table)
    path = Path(path)
    if format == "text":
        path.write_text(_text_of(table, kind))
        return
    payload = head + np.ascontiguousarray(block, dtype="<f8").tobytes()
    path.write_bytes(_HEAD.pack(MAGIC, VERSION, kind, degree) + payload + _CRC.pack(zlib.crc32(payload) & 0xFFFFFFFF))


def _text_of(table, kind: int) -> str:
    g = lambda x: format(float(x), ".17g")  # noqa: E731
    lines = [f"# ARVT v{VERSION} {_KIND_WORD[kind]}"]
    if kind == KIND_CONSTANT:
        lines += [f"# q = {table.q}", f"# construction = {table.construction}"]
        block = table.values
    elif kind == KIND_DYADIC:
        lines += [f"# degree = {table.degree}", f"# intervals = {table.n_intervals}", f"# decay = {g(table.decay)}"]
        block = table.coeffs
    elif kind == KIND_NCCHI2:
        lower, upper = _ncchi2_halves(table)
        decay = table.lower[0].decay if hasattr(table, "lower") else 0.5
        lines += [f"# nu = {g(table.nu)}", f"# knots = {table.n_knots}", f"# degree = {table.degree}",
                  f"# intervals = {table.n_intervals}", f"# decay = {g(decay)}"]
        block = np.concatenate([lower.reshape(-1), upper.reshape(-1)])
    else:
        lines += [f"# degree = {table.degree}", f"# octaves = {table.n_octaves}", f"# sub_bits = {table.sub_bits}"]
        block = table.coeffs
    lines += [g(v) for v in np.asarray(block, dtype=np.float64).reshape(-1)]
    return "\n".join(lines) + "\n"


def import_table(path):
    """Read a binary or text ARVT file; returns this package's table types."""
    path = Path(path)
    data = path.read_bytes()
    if data.startswith(b"# ARVT"):
        return _parse_text(data.decode("utf-8"))
    if data[:4] != MAGIC:
        raise BadMagicError(f"{path}: not a table file (bad magic)")
    if len(data) < _HEAD.size + _CRC.size:
        raise TruncatedFileError(f"{path}: too short for header and checksum")
    _, version, kind, degree = _HEAD.unpack_from(data, 0)
    if version != VERSION:
        raise VersionError(f"{path}: format version {version} not supported (expected {VERSION})")
    payload = data[_HEAD.size:-_CRC.size]
    if (zlib.crc32(payload) & 0xFFFFFFFF) != _CRC.unpack_from(data, len(data) - _CRC.size)[0]:
        raise ChecksumError(f"{path}: payload CRC-32 mismatch")
    fields = _FIELDS.get(kind)
    if fields is None:
        raise TableIOError(f"unknown table kind code {kind}")
    if len(payload) < fields.size:
        raise TruncatedFileError("file ended inside a header field")
    head = fields.unpack_from(payload, 0)
    block = payload[fields.size:]

    def coeffs(count: int) -> np.ndarray:
        if len(block) < 8 * count:
            raise TruncatedFileError(f"file ended inside the coefficient block ({len(block)} of {8 * count} bytes)")
        return np.frombuffer(block, dtype="<f8", count=count).astype(np.float64)

    if kind == KIND_CONSTANT:
        q, cons = head
        if cons >= len(CONSTRUCTIONS):
            raise TableIOError(f"unknown construction code {cons}")
        return ConstantTable(q, coeffs(1 << q), CONSTRUCTIONS[cons])
    if kind == KIND_DYADIC:
        k, decay = head
        return DyadicPolyTable(degree, k, coeffs((degree + 1) * (k + 1)).reshape(degree + 1, k + 1), decay)
    if kind == KIND_NCCHI2:
        nu, n_knots, k, _decay = head
        both = coeffs(2 * n_knots * (degree + 1) * (k + 1)).reshape(2, n_knots, degree + 1, k + 1)
        return NcChi2Table.from_stacks(nu, np.stack([both[1], both[0]]))
    n_oct, sub_bits = head
    return SubDyadicTable(degree, n_oct, sub_bits,
                          coeffs((degree + 1) * n_oct << sub_bits).reshape(degree + 1, n_oct, 1 << sub_bits))


def _parse_text(text: str):
    lines = [ln.strip() for ln in text.splitlines() if ln.strip()]
    head = lines[0].split()
    if len(head) < 4 or head[1] != "ARVT":
        raise BadMagicError("not a text table file")
    if head[2] != f"v{VERSION}":
        raise VersionError(f"text format version {head[2]} not supported")
    meta, vals = {}, []
    for ln in lines[1:]:
        if ln.startswith("#"):
            key, _, val = ln[1:].partition("=")
            meta[key.strip()] = val.strip()
        else:
            vals.append(ln)
    try:
        arr = np.array([float(v) for v in vals], dtype=np.float64)
        kind = head[3]
        if kind == "constant":
            return ConstantTable(int(meta["q"]), arr, meta["construction"])
        if kind == "dyadic":
            m, k = int(meta["degree"]), int(meta["intervals"])
            return DyadicPolyTable(m, k, arr.reshape(m + 1, k + 1), float(meta["decay"]))
        if kind == "ncchi2":
            m, k, nk = int(meta["degree"]), int(meta["intervals"]), int(meta["knots"])
            if arr.size != 2 * nk * (m + 1) * (k + 1):
                raise TruncatedFileError(f"expected {2 * nk * (m + 1) * (k + 1)} coefficients, found {arr.size}")
            both = arr.reshape(2, nk, m + 1, k + 1)
            return NcChi2Table.from_stacks(float(meta["nu"]), np.stack([both[1], both[0]]))
        if kind == "subdyadic":
            m, no, sb = int(meta["degree"]), int(meta["octaves"]), int(meta["sub_bits"])
            return SubDyadicTable(m, no, sb, arr.reshape(m + 1, no, 1 << sb))
    except KeyError as exc:
        raise TableIOError(f"text table missing metadata field {exc}") from exc
    except ValueError as exc:
        raise TruncatedFileError(f"coefficient block malformed: {exc}") from exc
    raise TableIOError(f"unknown text table kind {head[3]!r}")
