"""PQZ1 / PQL1 / IVF1 persistence: files written by the
real reference (tests/golden/make_golden.py, g_formats) load to the same
arrays, our writers reproduce them byte for byte, and malformed input raises
FormatError with the byte offset (_binio.py:11-18).  CPU only."""

import os

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from paper_1712_02912_b200 import formats as F
from tests.conftest import GOLDEN


def _path(name):
    return os.path.join(GOLDEN, name)


def test_load_reference_files(golden):
    g = golden("formats.npz")
    pq8 = P.load_quantizer(_path("fmt_pq8.pqz"))
    np.testing.assert_array_equal(pq8.codebooks, g["pq8_books"])
    assert (pq8.m, pq8.b, pq8.d) == (4, 8, 32)
    cl8, b8 = P.load_codes(_path("fmt_codes8.pql"))
    assert b8 == 8
    np.testing.assert_array_equal(cl8.codes, g["codes8"])
    np.testing.assert_array_equal(cl8.ids, g["ids8"])
    cl4, b4 = P.load_codes(_path("fmt_codes4.pql"))
    assert b4 == 4
    np.testing.assert_array_equal(cl4.codes, g["codes4"])
    np.testing.assert_array_equal(cl4.ids, np.arange(g["codes4"].shape[0]))
    cl3, b3 = P.load_codes(_path("fmt_codes3.pql"))
    assert b3 == 3 and cl3.m == 5
    np.testing.assert_array_equal(cl3.codes, g["codes3"])
    idx = P.load_ivf(_path("fmt_index.ivf"))
    np.testing.assert_array_equal(idx.coarse, g["ivf_coarse"])
    np.testing.assert_array_equal(idx.pq.codebooks, g["ivf_books"])
    np.testing.assert_array_equal([l.n for l in idx.lists], g["ivf_sizes"])
    np.testing.assert_array_equal(np.concatenate([l.codes for l in idx.lists]), g["ivf_codes"])
    np.testing.assert_array_equal(np.concatenate([l.ids for l in idx.lists]), g["ivf_ids"])


@pytest.mark.parametrize("name", ["fmt_pq8.pqz", "fmt_pq4.pqz", "fmt_codes8.pql", "fmt_codes4.pql",
                                  "fmt_codes3.pql", "fmt_index.ivf"])
def test_writers_byte_identical(tmp_path, name):
    src = _path(name)
    out = tmp_path / name
    if name.endswith(".pqz"):
        P.save_quantizer(out, P.load_quantizer(src))
    elif name.endswith(".pql"):
        cl, b = P.load_codes(src)
        P.save_codes(out, cl, b)
    else:
        P.save_ivf(out, P.load_ivf(src))
    assert out.read_bytes() == open(src, "rb").read()


def test_format_errors(tmp_path):
    raw = open(_path("fmt_codes8.pql"), "rb").read()
    bad = tmp_path / "bad.pql"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(P.FormatError) as e:
        P.load_codes(bad)
    assert e.value.offset == 0 and isinstance(e.value, ValueError)
    bad.write_bytes(raw[:100])
    with pytest.raises(P.FormatError) as e:
        P.load_codes(bad)
    assert e.value.offset == 20     # the code payload starts after 4 + 4 x 4 header bytes
    bad.write_bytes(raw[:10])
    with pytest.raises(P.FormatError):
        P.load_codes(bad)
    with pytest.raises(ValueError):
        P.save_codes(tmp_path / "x.pql", P.CodeList(np.full((3, 2), 16, np.uint8)), 4)


def test_pack_roundtrip():
    rng = np.random.default_rng(1)
    for m in (1, 2, 5, 16):
        c = rng.integers(0, 16, (37, m)).astype(np.uint8)
        np.testing.assert_array_equal(F.unpack_codes(F.pack_codes(c, 4).reshape(-1), 37, m, 4), c)
