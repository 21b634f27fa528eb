"""PQ Fast Scan (fastscan.py) -- CPU side: the oracle's
sequential pruned scan and its ScanStats against the reference's outputs
(tests/golden/fastscan.npz), the grouped container (group_codes, pack_code,
group_key, relabel_codes) and PQG1 files written by the reference."""

import io
import os

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from paper_1712_02912_b200 import fastscan as F
from tests.conftest import GOLDEN

SETTINGS = [(0.01, 100), (0.05, 10), (0.001, 1), (1.0, 50), (0.0002, 300)]


@pytest.mark.parametrize("init,r", SETTINGS)
def test_oracle_fast_scan_golden(golden, init, r):
    g = golden("fastscan.npz")
    order = O.group_order(g["codes"])
    codes, ids = g["codes"][order], g["ids"][order]
    tag = f"i{init}_r{r}"
    for qi, q in enumerate(g["queries"]):
        d, i, checked, pruned = O.fast_scan(codes, ids, O.compute_tables(g["codebooks"], q), init, r)
        n = len(d)
        np.testing.assert_array_equal(d, g[f"{tag}_dist"][qi][:n])
        np.testing.assert_array_equal(i, g[f"{tag}_ids"][qi][:n])
        assert (codes.shape[0], checked, pruned) == tuple(g[f"{tag}_stats"][qi])
        # exact: the same set as the exhaustive scan
        sd, si = O.scan(codes, ids, O.compute_tables(g["codebooks"], q), r)
        np.testing.assert_array_equal(sd, d)
        np.testing.assert_array_equal(si, i)


def test_group_codes_golden(golden):
    g = golden("fastscan.npz")
    gr = F.group_codes(P.CodeList(g["codes"], g["ids"]))
    for k in ("keys", "offsets", "counts", "packed", "ids"):
        np.testing.assert_array_equal(getattr(gr, k), g[f"g_{k}"])
    np.testing.assert_array_equal(gr.reconstruct_codes(), g["codes"][O.group_order(g["codes"])])
    c = g["codes"][5]
    np.testing.assert_array_equal(F.pack_code(c), g["g_packed"][list(gr.ids).index(g["ids"][5])])
    assert F.group_key(c) == tuple(int(v) >> 4 for v in c[:4])


def test_grouped_validation():
    gr = F.group_codes(P.CodeList(np.arange(80, dtype=np.uint8).reshape(10, 8)))
    with pytest.raises(ValueError):
        F.GroupedDatabase(gr.keys, gr.offsets + 1, gr.counts, gr.packed, gr.ids)
    with pytest.raises(ValueError):
        F.GroupedDatabase(gr.keys, gr.offsets, gr.counts, gr.packed[:-1], gr.ids)
    with pytest.raises(ValueError):
        F.group_codes(P.CodeList(np.zeros((4, 4), np.uint8)))


def test_relabel_codes():
    rng = np.random.default_rng(0)
    perm = np.stack([rng.permutation(256) for _ in range(8)])
    codes = rng.integers(0, 256, (100, 8)).astype(np.uint8)
    out = F.relabel_codes(codes, perm)
    for j in range(8):
        assert np.all(perm[j][out[:, j]] == codes[:, j])


def test_pqg1_reference_file_roundtrip(golden):
    path = os.path.join(GOLDEN, "fmt_grouped.pqg")
    gr = F.load_grouped(path)
    g = golden("fastscan.npz")
    want = F.group_codes(P.CodeList(g["codes"][:300], g["ids"][:300]))
    for k in ("keys", "offsets", "counts", "packed", "ids"):
        np.testing.assert_array_equal(getattr(gr, k), getattr(want, k))
    buf = io.BytesIO()
    F.write_grouped_body(buf, gr)
    assert buf.getvalue() == open(path, "rb").read()
    with pytest.raises(P.FormatError):
        F.read_grouped_body(io.BytesIO(open(path, "rb").read()[:40]))
    with pytest.raises(P.FormatError):
        F.read_grouped_body(io.BytesIO(b"PQL1" + open(path, "rb").read()[4:]))
