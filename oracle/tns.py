"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's .tns reader
(read_tns, /root/reference/proj/src/io.cpp:42-126), the checker for the GPU
reader (qd_read_tns).  Pinned against the reference's own read_tns through
oracle/_ref (tests/test_tns.py).  Never imported by the product.

* lines: std::getline on '\\n' (io.cpp:55) — a final line without '\\n' counts,
  a trailing '\\n' does not start another line;
* fields: split on ' ', '\\t', '\\r' (io.cpp:22-34); blank lines and lines whose
  first field starts with '#' are skipped (io.cpp:57);
* the first data line fixes the field count (io.cpp:59-72);
* indices: std::from_chars(uint32_t), 1-based (io.cpp:82-100);
* values: std::from_chars(double) (io.cpp:108-113) — grammar below, correctly
  rounded (Python float() is), overflow to inf / underflow to 0 rejected
  (libstdc++ returns result_out_of_range; measured with g++ 13 here);
* dims: declared, else the per-mode maximum 1-based index (io.cpp:115-124);
  check_valid (coo.cpp:8-30); canonicalise = stable sort by all modes
  (io.cpp:36-38).
"""
from __future__ import annotations

import re
import struct

import numpy as np

_DEC = re.compile(rb"-?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?")
_INF = re.compile(rb"-?(?:inf|infinity)", re.I)
_NAN = re.compile(rb"-?nan(?:\([A-Za-z0-9_]*\))?", re.I)
_IDX = re.compile(rb"[0-9]+")


class TnsParseError(Exception):
    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


class TnsInvalid(Exception):
    pass


def from_chars_f64(tok: bytes):
    """std::from_chars(double) over the whole token; None when rejected."""
    neg = tok.startswith(b"-")
    if _INF.fullmatch(tok):
        return -np.inf if neg else np.inf
    if _NAN.fullmatch(tok):
        bits = (1 << 63 if neg else 0) | 0x7FF8000000000000
        return struct.unpack("<d", struct.pack("<Q", bits))[0]
    if not _DEC.fullmatch(tok):
        return None
    v = float(tok.decode())
    mant = tok.split(b"e")[0].split(b"E")[0]
    nonzero = any(c in b"123456789" for c in mant)
    if v in (np.inf, -np.inf) or (v == 0.0 and nonzero):
        return None
    return v


def from_chars_u32(tok: bytes):
    if not _IDX.fullmatch(tok):
        return None
    v = int(tok)
    return v if v <= 0xFFFFFFFF else None


def read_tns_bytes(text: bytes, declared_dims=None, canonicalize: bool = True):
    """Returns (dims u32[r], coords u32[N*r], values f64[N]) or raises
    TnsParseError / TnsInvalid like io.cpp / coo.cpp."""
    lines = text.split(b"\n")
    if text.endswith(b"\n") or not text:
        lines = lines[:-1]
    decl = None if declared_dims is None else [int(d) for d in declared_dims]
    F = 0
    coords, values = [], []
    max_index = []
    lineno = 0
    for raw in lines:
        lineno += 1
        fields = [f for f in re.split(rb"[ \t\r]+", raw) if f]
        if not fields or fields[0].startswith(b"#"):
            continue
        if F == 0:
            if len(fields) < 2:
                raise TnsParseError(lineno, "expected at least one index and a value, got "
                                    f"{len(fields)} fields")
            if decl is not None and len(decl) != len(fields) - 1:
                raise TnsParseError(lineno, f"file has rank {len(fields) - 1} but {len(decl)} "
                                    "dimensions were declared")
            F = len(fields)
            max_index = [0] * (F - 1)
        elif len(fields) != F:
            raise TnsParseError(lineno, f"expected {F} fields, got {len(fields)}")
        for m in range(F - 1):
            tok = fields[m]
            idx = from_chars_u32(tok)
            t = tok.decode("latin-1")
            if idx is None:
                raise TnsParseError(lineno, f"invalid index '{t}'")
            if idx < 1:
                raise TnsParseError(lineno, f"indices are 1-based; got {t} in mode {m + 1}")
            if decl is not None and idx > decl[m]:
                raise TnsParseError(lineno, f"index {t} exceeds declared dimension {decl[m]} "
                                    f"of mode {m + 1}")
            max_index[m] = max(max_index[m], idx)
            coords.append(idx - 1)
        v = from_chars_f64(fields[-1])
        if v is None:
            raise TnsParseError(lineno, f"invalid value '{fields[-1].decode('latin-1')}'")
        values.append(v)
    if F == 0:
        if decl is None:
            raise TnsParseError(lineno, "empty file: rank is unknowable without declared "
                                "dimensions")
        dims = decl
    else:
        dims = decl if decl is not None else max_index
    r = len(dims)
    if r == 0:
        raise TnsInvalid("tensor rank must be positive")
    for m, d in enumerate(dims):
        if d == 0:
            raise TnsInvalid(f"dimension of mode {m} must be positive")
    c = np.asarray(coords, np.uint32).reshape(-1, r)
    v = np.asarray(values, np.float64)
    if canonicalize and len(v) > 1:
        order = np.lexsort(tuple(c[:, m] for m in reversed(range(r))))  # stable
        c, v = c[order], v[order]
    return np.asarray(dims, np.uint32), np.ascontiguousarray(c).reshape(-1), v


def _fmt_value(x: float) -> str:
    """std::to_chars(double), shortest round-trip (io.cpp:145): Python's repr
    gives the same shortest digits; the layout (fixed vs scientific, the
    shorter, fixed on a tie; exact digits for integer values; 2-digit
    exponents) is restated here."""
    if x != x:
        neg = struct.unpack("<Q", struct.pack("<d", x))[0] >> 63
        return "-nan" if neg else "nan"
    if x in (np.inf, -np.inf):
        return "inf" if x > 0 else "-inf"
    sign = "-" if struct.unpack("<Q", struct.pack("<d", x))[0] >> 63 else ""
    x = abs(x)
    if x == 0.0:
        return sign + "0"
    r = repr(x)  # shortest round-trip digits
    mant, _, exp = r.partition("e")
    e = int(exp) if exp else 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    lead_zeros = len(ip + fp) - len((ip + fp).lstrip("0"))
    X = len(ip) - 1 + e - lead_zeros  # scientific exponent of the first digit
    digits = digits.rstrip("0") or "0"
    n = len(digits)
    ax = abs(X)
    sci = n + (1 if n > 1 else 0) + 2 + (3 if ax >= 100 else 2)
    if X >= n - 1:
        fix = X + 1
    elif X >= 0:
        fix = n + 1
    else:
        fix = n + 1 - X
    if fix <= sci:
        if X >= n - 1:
            return sign + str(int(x))  # exact integer digits
        if X >= 0:
            return sign + digits[:X + 1] + "." + digits[X + 1:]
        return sign + "0." + "0" * (-X - 1) + digits
    s = digits[0] + ("." + digits[1:] if n > 1 else "")
    return f"{sign}{s}e{'-' if X < 0 else '+'}{ax:02d}"


def write_tns_bytes(dims, coords, values) -> bytes:
    """write_tns (io.cpp:128-152): storage order, 1-based indices (u32
    arithmetic, so 2^32-1 + 1 wraps to 0), ' '-separated, '\n' per row."""
    r = len(dims)
    c = np.asarray(coords, np.uint32).reshape(-1, r) if r else np.zeros((0, 0), np.uint32)
    out = []
    for row, v in zip(c, np.asarray(values, np.float64)):
        idx = " ".join(str((int(x) + 1) & 0xFFFFFFFF) for x in row)
        out.append(f"{idx} {_fmt_value(float(v))}\n")
    return "".join(out).encode()
