"""Derived quantizers (derived.py) -- CPU side: the oracle's
two-pass search and query_ivf(kernel='derived') against the reference's
outputs (tests/golden/derived.npz), and the PQZ1+derived / IVF1+derived files
the reference wrote (load, byte-identical rewrite)."""

import io
import os

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from paper_1712_02912_b200 import derived as D
from paper_1712_02912_b200 import formats as F
from tests.conftest import GOLDEN

SETTINGS = [(10, 50), (100, 9000), (5, 1), (20, 300), (50, 6000)]
IVF_SETTINGS = [(3, 20, 100), (12, 50, None), (2, 10, 1)]


@pytest.mark.parametrize("r,r2", SETTINGS)
def test_oracle_two_pass_golden(golden, r, r2):
    g = golden("derived.npz")
    for qi, q in enumerate(g["queries"]):
        d, i = O.search_two_pass(g["books"], g["derived"], g["codes"], g["ids"], q, r, r2)
        n = len(d)
        np.testing.assert_array_equal(d, g[f"r{r}_r2{r2}_dist"][qi][:n])
        np.testing.assert_array_equal(i, g[f"r{r}_r2{r2}_ids"][qi][:n])
        assert np.all(g[f"r{r}_r2{r2}_ids"][qi][n:] == -1)


def ivf_lists(g):
    offs = np.concatenate([[0], np.cumsum(g["ivf_sizes"])])
    codes = [g["ivf_codes"][offs[c]:offs[c + 1]] for c in range(len(g["ivf_sizes"]))]
    ids = [g["ivf_ids"][offs[c]:offs[c + 1]] for c in range(len(g["ivf_sizes"]))]
    return codes, ids


@pytest.mark.parametrize("ma,r,r2", IVF_SETTINGS)
def test_oracle_ivf_derived_golden(golden, ma, r, r2):
    g = golden("derived.npz")
    codes, ids = ivf_lists(g)
    rr2 = r2 if r2 is not None else P.default_r2(r)
    for qi, q in enumerate(g["queries"]):
        d, i = O.query_ivf_derived(g["ivf_coarse"], g["ivf_books"], g["ivf_derived"], codes, ids, q, ma, r, rr2)
        n = len(d)
        np.testing.assert_array_equal(d, g[f"ivf_ma{ma}_r{r}_r2{r2}_dist"][qi][:n])
        np.testing.assert_array_equal(i, g[f"ivf_ma{ma}_r{r}_r2{r2}_ids"][qi][:n])


def test_derived_files(golden, tmp_path):
    g = golden("derived.npz")
    path = os.path.join(GOLDEN, "fmt_derived.pqz")
    dpq = P.load_quantizer_any(path)
    assert isinstance(dpq, D.DerivedPQ) and dpq.bbar == 4
    np.testing.assert_array_equal(dpq.derived, g["derived"])
    np.testing.assert_array_equal(dpq.pq.codebooks, g["books"])
    buf = io.BytesIO()
    D.write_derived_body(buf, dpq)
    assert buf.getvalue() == open(path, "rb").read()
    assert not isinstance(P.load_quantizer_any(os.path.join(GOLDEN, "fmt_pq8.pqz")), D.DerivedPQ)
    ipath = os.path.join(GOLDEN, "fmt_index_derived.ivf")
    idx = P.load_ivf(ipath)
    assert idx.dpq is not None and idx.dpq.pq is idx.pq and idx.dpq.bbar == 2 and idx.K == 4
    out = str(tmp_path / "index_derived.ivf")
    P.save_ivf(out, idx)
    assert open(out, "rb").read() == open(ipath, "rb").read()


def test_derived_validation():
    pq = P.ProductQuantizer(2, 4, 4, np.zeros((2, 16, 2), np.float32))
    with pytest.raises(ValueError):
        D.DerivedPQ(pq, 5, np.zeros((2, 32, 2), np.float32))
    with pytest.raises(ValueError):
        D.DerivedPQ(pq, 2, np.zeros((2, 8, 2), np.float32))
    dpq = D.DerivedPQ(pq, 2, np.zeros((2, 4, 2), np.float32))
    assert dpq.kbar == 4 and dpq.low_bits(13) == 1
    other = P.ProductQuantizer(2, 4, 4, np.zeros((2, 16, 2), np.float32))
    with pytest.raises(ValueError):
        P.IvfIndex(np.zeros((1, 4), np.float32), other, [P.CodeList(np.zeros((0, 2), np.uint8))], dpq=dpq)
