"""Edge-list ingestion (graph.py:152-209): the native multithreaded parser
(csrc/ingest.cu) against the reference's line loop, on CPU (host-only code)."""

import io

import numpy as np
import pytest

from paper_1708_07481_b200 import graph as G


def _same(native, python):
    s0, d0, w0, m0 = native
    s1, d1, w1, m1 = python
    assert np.array_equal(s0, s1) and np.array_equal(d0, d1) and m0 == m1
    assert (w0 is None) == (w1 is None)
    if w0 is not None:
        assert np.array_equal(w0, w1, equal_nan=True)


CASES = [
    b"1\t2\n2\t3\t0.5\n# comment\n\n3 1\n",
    b"",
    b"# only a comment\n",
    b"   \n\t\n",
    b"1 2",
    b"1 2\r\n3 4\r\n",
    b"+1 2 inf\n2 1 -0.0\n3 3 nan\n",
    b"5 7 1e-3\n7 5 2.5E+1\n5 5 .5\n6 6 5.\n",
    b"  #indented comment\n1 1\n",
    b"0007 0008 1\n",
    b"1\x0b2\x0c3\n",
]
ERRORS = [
    (b"1 2 3 4\n", "ParseError"),
    (b"1\n", "ParseError"),
    (b"a b\n", "ParseError"),
    (b"0 1\n", "ParseError"),       # below base 1
    (b"1 2 -1\n", "DomainError"),
    (b"1 2\n2 x\n", "ParseError"),
    (b"1 2 #c\n", "ParseError"),
    (b"\xc3\xa9 1\n", "ParseError"),
]


@pytest.mark.parametrize("data", CASES)
@pytest.mark.parametrize("base", [0, 1])
def test_native_matches_reference_loop(data, base):
    py = G._parse_python(io.BytesIO(data), base)
    nat = G._parse_native(data, base)
    if nat is None:  # outside the fast path: the loop decides (base 0/1 edge)
        return
    _same(nat, py)


@pytest.mark.parametrize("data,exc", ERRORS)
def test_errors_come_from_reference_rules(data, exc):
    assert G._parse_native(data, 1) is None
    with pytest.raises(Exception) as ei:
        G._parse_python(io.BytesIO(data), 1)
    assert type(ei.value).__name__ == exc


def test_underscores_and_unicode_fall_back():
    # int('1_0') == 10 in Python: the native path defers, the loop accepts
    data = b"1_0 2\n"
    assert G._parse_native(data, 1) is None
    s, d, w, m = G._parse_python(io.BytesIO(data), 1)
    assert s.tolist() == [9] and d.tolist() == [1]


@pytest.mark.parametrize("threads", [1, 3, 8, 0])
def test_chunked_parse_is_file_order(threads):
    rng = np.random.default_rng(0)
    m = 200_000
    s = rng.integers(1, 10_000, m)
    d = rng.integers(1, 10_000, m)
    w = rng.random(m)
    lines = [f"{a}\t{b}\t{float(x)!r}" if i % 7 else f"{a} {b}" for i, (a, b, x) in enumerate(zip(s, d, w))]
    lines.insert(50_000, "# mid comment")
    data = ("\n".join(lines) + "\n").encode()
    L = G.N.lib()
    m_, mx, hw, bad = G.N.C.c_int64(0), G.N.C.c_int64(0), G.N.C.c_int32(0), G.N.C.c_int64(0)
    h = G.N.C.c_void_p()
    assert L.spb_edge_list_parse(data, len(data), 1, threads, G.N.C.byref(m_), G.N.C.byref(mx),
                                 G.N.C.byref(hw), G.N.C.byref(bad), G.N.C.byref(h)) == 0
    src = np.empty(m_.value, np.int64)
    dst = np.empty(m_.value, np.int64)
    wt = np.empty(m_.value, np.float64)
    assert L.spb_edge_list_fetch(h, src.ctypes.data, dst.ctypes.data, wt.ctypes.data) == 0
    _same((src, dst, wt, mx.value), G._parse_python(io.BytesIO(data), 1))


def test_error_line_number_is_first_bad_line():
    good = b"1 2\n" * 100_000
    data = good + b"1 2 3 4\n" + good + b"x y\n"
    L = G.N.lib()
    m_, mx, hw, bad = G.N.C.c_int64(0), G.N.C.c_int64(0), G.N.C.c_int32(0), G.N.C.c_int64(0)
    h = G.N.C.c_void_p()
    st = L.spb_edge_list_parse(data, len(data), 1, 8, G.N.C.byref(m_), G.N.C.byref(mx),
                               G.N.C.byref(hw), G.N.C.byref(bad), G.N.C.byref(h))
    assert st == G.N.E_PARSE and bad.value == 100_001
