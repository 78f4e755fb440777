"""The .tns reader (read_tns, io.cpp:42-126) on the GPU (qd_read_tns).

CPU (not gpu): the Python restatement (oracle/tns.py) is pinned against the
reference's own read_tns (oracle/_ref, the unmodified io.cpp) on every case
below, and the device token parsers (tns_parse.cuh, compiled as host code) are
checked against std::from_chars on random and adversarial tokens.
GPU: qd_read_tns against the pinned restatement — same rows bit for bit, or
the same ParseError text and line.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

import tns as otns
from pyoracle import Reference, reference_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _random_text(rng, n, dims, fmt="repr", shuffle=True, dup=0.0):
    r = len(dims)
    c = np.stack([rng.integers(1, d + 1, n) for d in dims], 1)
    if dup:
        k = int(n * dup)
        c[rng.integers(0, n, k)] = c[rng.integers(0, n, k)]
    v = rng.random(n).tolist()
    if fmt == "exp":
        vals = [f"{x:.20e}" for x in v]
    elif fmt == "mixed":
        vals = [repr(x) if i % 3 else f"{x * 10.0 ** int(rng.integers(-300, 300)):.17g}"
                for i, x in enumerate(v)]
    else:
        vals = [repr(x) for x in v]
    lines = [" ".join(str(int(x)) for x in row) + " " + s for row, s in zip(c, vals)]
    if not shuffle:
        lines.sort()
    return ("\n".join(lines) + "\n").encode()


def cases():
    rng = np.random.default_rng(7)
    out = [
        ("basic", b"1 1 1 1.5\n2 1 3 -2\n1 2 1 0.25\n", None, True),
        ("comments_blank_crlf_tabs",
         b"# header\n\n1\t2 3\t0.5\r\n   # indented comment\n2 2 2 7e-3\r\n\t\n3 1 1 -0\n", None,
         True),
        ("no_final_newline", b"1 1 1.0\n2 3 2.0", None, True),
        ("raw_order", b"3 1 1\n1 2 2\n2 1 3\n1 1 4\n", None, False),
        ("declared", b"1 1 1\n2 2 2\n", [5, 7], True),
        ("declared_empty_ok", b"# nothing\n\n", [3, 4, 5], True),
        ("values_special",
         b"1 inf\n2 -Infinity\n3 nan\n4 -nan\n5 NaN(abc_1)\n6 5.\n7 .5\n8 -0.0\n"
         b"9 4.9e-324\n10 1.7976931348623157e308\n11 2.2250738585072011e-308\n"
         b"12 9007199254740993.0000000000000000000000000001\n13 1E+5\n14 00012\n"
         b"15 0e99999\n16 2.4703282292062328e-324\n", None, False),
        ("leading_zero_index", b"0001 02 3\n", None, True),
        ("duplicates_stable", b"2 1 1\n1 1 2\n2 1 3\n1 1 4\n2 1 5\n", None, True),
        # errors
        ("err_first_line_one_field", b"# c\n5\n1 2\n", None, True),
        ("err_rank_vs_declared", b"\n1 2 3 4\n", [3, 3], True),
        ("err_field_count", b"1 1 1\n1 2 2\n1 2\n", None, True),
        ("err_field_count_more", b"1 1 1\n1 2 2 2 2\n", None, True),
        ("err_invalid_index", b"1 1 1\n1 1a 2\n", None, True),
        ("err_plus_index", b"+1 1 1\n", None, True),
        ("err_negative_index", b"-1 1 1\n", None, True),
        ("err_index_overflow", b"4294967296 1 1\n", None, True),
        ("err_zero_index", b"1 1 1\n2 0 1\n", None, True),
        ("err_exceeds_declared", b"1 1 1\n2 9 1\n", [4, 4], True),
        ("err_value_junk", b"1 1 1.0x\n", None, True),
        ("err_value_exponent", b"1 1 1e\n", None, True),
        ("err_value_plus", b"1 1 +1\n", None, True),
        ("err_value_overflow", b"1 1 1\n1 2 1e400\n", None, True),
        ("err_value_underflow", b"1 1 1e-400\n", None, True),
        ("err_value_underflow_halfway", b"1 1 2.4703282292062327e-324\n", None, True),
        ("err_value_hex", b"1 1 0x10\n", None, True),
        ("err_value_nan_open", b"1 1 nan(\n", None, True),
        ("err_value_infin", b"1 1 infin\n", None, True),
        ("err_empty_file", b"", None, True),
        ("err_comment_only", b"# only\n\n#x\n", None, True),
        ("err_first_error_wins", b"1 1 1\n1 1 x\n1 0 1\n1 1\n", None, True),
        ("invalid_declared_zero_dim", b"\n", [3, 0], True),
        ("invalid_declared_rank0", b"", [], True),
    ]
    out.append(("random_r3", _random_text(rng, 3000, [40, 30, 50]), None, True))
    out.append(("random_r4_dups", _random_text(rng, 4000, [9, 8, 7, 6], dup=0.3), None, True))
    out.append(("random_r2_exp", _random_text(rng, 2000, [1000, 3], fmt="exp"), None, False))
    out.append(("random_mixed_declared", _random_text(rng, 2500, [20, 20, 20], fmt="mixed"),
                [20, 20, 25], True))
    # hard decimal -> double: 17-40 digit neighbours of halfway points
    hard = []
    for i in range(600):
        x = float(rng.random() * 10.0 ** int(rng.integers(-320, 300)))
        if x == 0.0:
            continue
        nxt = np.nextafter(x, np.inf)
        mid = (np.longdouble(x) + np.longdouble(nxt)) / 2
        s = np.format_float_scientific(mid, precision=int(rng.integers(17, 40)), unique=False)
        hard.append(f"{i + 1} {s}")
    out.append(("halfway_values", ("\n".join(hard) + "\n").encode(), None, False))
    return out


CASES = cases()
IDS = [c[0] for c in CASES]


def _oracle(text, decl, canon):
    try:
        return ("ok",) + otns.read_tns_bytes(text, decl, canon)
    except otns.TnsParseError as e:
        return ("parse", str(e), e.line)
    except otns.TnsInvalid as e:
        return ("invalid", str(e))


def _same_rows(a, b):
    return (np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
            and np.array_equal(np.asarray(a[3]).view(np.uint64), np.asarray(b[3]).view(np.uint64)))


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,text,decl,canon", CASES, ids=IDS)
def test_oracle_matches_reference_read_tns(tmp_path, name, text, decl, canon):
    p = tmp_path / "t.tns"
    p.write_bytes(text)
    want = _oracle(text, decl, canon)
    try:
        got = ("ok",) + Reference().read_tns(p, decl, canon)
    except Exception as e:  # OracleError
        if getattr(e, "code", 0) == 4:
            got = ("parse", str(e).split(": ", 1)[1], e.line)
        else:
            got = ("invalid", str(e).split(": ", 1)[1])
    assert got[0] == want[0], (got, want)
    if want[0] == "ok":
        assert _same_rows(got, want)
    else:
        assert got[1:] == want[1:]


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_oracle_reads_reference_write_tns(tmp_path):
    rng = np.random.default_rng(11)
    dims = np.array([50, 60, 70], np.uint32)
    c = np.stack([rng.integers(0, d, 2000) for d in dims], 1).astype(np.uint32).reshape(-1)
    v = rng.standard_normal(2000) * 10.0 ** rng.integers(-200, 200, 2000)
    p = tmp_path / "w.tns"
    Reference().write_tns(dims, c, v, p)
    d2, c2, v2 = otns.read_tns_bytes(p.read_bytes(), None, False)
    assert np.array_equal(c2, c) and np.array_equal(v2.view(np.uint64), v.view(np.uint64))


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_device_token_parsers_match_from_chars(tmp_path):
    exe = tmp_path / "tpc"
    subprocess.run(["g++", "-O2", "-std=c++20", "-I",
                    os.path.join(ROOT, "paper_2005_10427_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "tns_parse_check.cpp"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe), "60000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-2000:]
    assert " 0 mismatches" in r.stdout


# ---- GPU ----------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name,text,decl,canon", CASES, ids=IDS)
def test_gpu_read_tns_matches_oracle(name, text, decl, canon):
    import paper_2005_10427_b200 as qb
    want = _oracle(text, decl, canon)
    try:
        t = qb.read_tns_text(text, decl, canon)
        got = ("ok", t.dims, t.coords, t.values)
    except qb.ParseError as e:
        got = ("parse", str(e), e.line())
    except qb.InvalidArgument as e:
        got = ("invalid", str(e))
    assert got[0] == want[0], (got, want)
    if want[0] == "ok":
        assert _same_rows(got, want)
    else:
        assert got[1:] == want[1:]


@pytest.mark.gpu
def test_gpu_read_tns_large(tmp_path):
    """300K lines (multiple line CTAs and text tiles), canonicalised on device."""
    import paper_2005_10427_b200 as qb
    rng = np.random.default_rng(5)
    text = _random_text(rng, 300_000, [3000, 200, 5000], fmt="mixed", dup=0.05)
    p = tmp_path / "big.tns"
    p.write_bytes(text)
    t = qb.read_tns(p)
    d, c, v = otns.read_tns_bytes(text, None, True)
    assert np.array_equal(t.dims, d) and np.array_equal(t.coords, c)
    assert np.array_equal(t.values.view(np.uint64), v.view(np.uint64))
    # error near the end of a big file: the first failing line wins
    bad = text[:-20] + b"\n1 1 1 oops\n1 0 1 2\n"
    with pytest.raises(qb.ParseError) as ei:
        qb.read_tns_text(bad)
    with pytest.raises(otns.TnsParseError) as eo:
        otns.read_tns_bytes(bad)
    assert str(ei.value) == str(eo.value) and ei.value.line() == eo.value.line


# ---- writer (write_tns, io.cpp:128-152) --------------------------------------

def _writer_cases():
    rng = np.random.default_rng(21)
    out = []
    n = 5000
    c = np.stack([rng.integers(0, d, n) for d in (70, 5, 900)], 1).astype(np.uint32)
    v = rng.random(n) * 10.0 ** rng.integers(-30, 30, n)
    out.append(("random", np.array([70, 5, 900], np.uint32), c.reshape(-1), v))
    bits = rng.integers(0, 2 ** 63, 20000, dtype=np.uint64) | (
        rng.integers(0, 2, 20000, dtype=np.uint64) << np.uint64(63))
    vb = bits.view(np.float64)
    out.append(("bit_patterns", np.array([20000], np.uint32),
                np.arange(20000, dtype=np.uint32), vb))
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, 0.1, 1e-4, 1e-3, 1e16, 1e21,
                        1.2345678901234567e21, 12300000.0, 5e-324, 1.7976931348623157e308,
                        2.0 ** 70, 2.0 ** -1074, 123456.0, 0.5, 2.0 / 3.0])
    out.append(("special", np.array([4294967295, 2], np.uint32),
                np.stack([np.arange(len(special)) * 200000000, np.arange(len(special)) % 2], 1)
                .astype(np.uint32).reshape(-1), special))
    out.append(("max_coord", np.array([4294967295], np.uint32),
                np.array([4294967294, 0], np.uint32), np.array([1.5, 2.5])))
    out.append(("empty", np.array([3, 3], np.uint32), np.zeros(0, np.uint32), np.zeros(0)))
    return out


WCASES = _writer_cases()


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_device_formatter_matches_to_chars(tmp_path):
    exe = tmp_path / "tfc"
    subprocess.run(["g++", "-O2", "-std=c++20", "-I",
                    os.path.join(ROOT, "paper_2005_10427_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "tns_format_check.cpp"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe), "200000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-2000:]
    assert " 0 mismatches" in r.stdout


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,dims,coords,values", WCASES, ids=[w[0] for w in WCASES])
def test_oracle_writer_matches_reference(tmp_path, name, dims, coords, values):
    p = tmp_path / "w.tns"
    Reference().write_tns(dims, coords, values, p)
    assert p.read_bytes() == otns.write_tns_bytes(dims, coords, values)


@pytest.mark.gpu
@pytest.mark.parametrize("name,dims,coords,values", WCASES, ids=[w[0] for w in WCASES])
def test_gpu_write_tns_matches_oracle(tmp_path, name, dims, coords, values):
    import paper_2005_10427_b200 as qb
    t = qb.CooTensor(dims, coords, values)
    want = otns.write_tns_bytes(dims, coords, values)
    assert qb.write_tns_text(t) == want
    p = tmp_path / "g.tns"
    qb.write_tns(t, p)
    assert p.read_bytes() == want


@pytest.mark.gpu
def test_gpu_write_read_round_trip():
    """write_tns -> read_tns returns the tensor (io.hpp:43-46), 200K rows."""
    import paper_2005_10427_b200 as qb
    rng = np.random.default_rng(3)
    dims = np.array([500, 40, 3000], np.uint32)
    n = 200_000
    c = np.stack([rng.integers(0, d, n) for d in dims], 1).astype(np.uint32)
    c[0] = dims - 1  # every dim reached, so the read-back dims match
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    t = qb.CooTensor(dims, c.reshape(-1), v)
    back = qb.read_tns_text(qb.write_tns_text(t), canonicalize=False)
    assert back == t


@pytest.mark.gpu
def test_gpu_read_tns_slow_path_list_overflow(monkeypatch):
    """Values that need the big-integer path are finished by k_line_slow from
    a bounded list; when the list overflows every line is re-parsed with the
    slow path inline.  Both give the oracle's rows."""
    import paper_2005_10427_b200 as qb
    name, text, decl, canon = [c for c in CASES if c[0] == "halfway_values"][0]
    want = _oracle(text, decl, canon)
    for cap in ("1000000", "4", "0"):
        monkeypatch.setenv("QD_TNS_SLOW_CAP", cap)
        t = qb.read_tns_text(text, decl, canon)
        assert _same_rows(("ok", t.dims, t.coords, t.values), want), cap
    # a slow-path value that underflows is still the first failing line
    bad = b"1 1.0\n2 2.47032822920623272088e-324\n3 x\n"
    monkeypatch.setenv("QD_TNS_SLOW_CAP", "8")
    with pytest.raises(qb.ParseError) as ei:
        qb.read_tns_text(bad)
    with pytest.raises(otns.TnsParseError) as eo:
        otns.read_tns_bytes(bad)
    assert str(ei.value) == str(eo.value) and ei.value.line() == 2
