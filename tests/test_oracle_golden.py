"""Pin the CPU oracle (oracle/pqscan_oracle.py) to fixtures produced by the
real reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import pqscan_oracle as O


@pytest.mark.parametrize("tag", ["c0", "c1", "c2"])
def test_tables_bitwise(golden, tag):
    g = golden("tables.npz")
    books, qs, tabs = g[f"{tag}_codebooks"], g[f"{tag}_queries"], g[f"{tag}_tables"]
    got = O.compute_tables_batch(books, qs)
    assert got.dtype == np.float32
    np.testing.assert_array_equal(got.view(np.uint32), tabs.view(np.uint32))


@pytest.mark.parametrize("tag", ["c0", "c1", "c2"])
def test_scan_distances_bitwise(golden, tag):
    g = golden("tables.npz")
    for qi in range(g[f"{tag}_tables"].shape[0]):
        got = O.scan_distances(g[f"{tag}_tables"][qi], g[f"{tag}_codes"])
        np.testing.assert_array_equal(got, g[f"{tag}_dist"][qi])


def test_scan_cases(golden):
    g = golden("scan.npz")
    for c in range(int(g["ncases"])):
        r = int(g[f"{c}_r"])
        d, i = O.scan(g[f"{c}_codes"], g[f"{c}_ids"], g[f"{c}_tables"], r)
        cnt = int(g[f"{c}_count"])
        assert len(d) == cnt
        np.testing.assert_array_equal(d, g[f"{c}_dist"][:cnt])
        np.testing.assert_array_equal(i, g[f"{c}_out_ids"][:cnt])


def test_quick_adc_settings(golden):
    g = golden("quick_adc.npz")
    codes, books, qs = g["codes"], g["codebooks"], g["queries"]
    ids = np.arange(codes.shape[0], dtype=np.int64)
    for s in range(6):
        init, r = int(g[f"s{s}_init"]), int(g[f"s{s}_r"])
        for qi, q in enumerate(qs):
            t = O.compute_tables(books, q)
            bins, oid, qt, qmin, qmax = O.qadc_scan(codes, ids, t, init, r)
            n = len(bins)
            np.testing.assert_array_equal(bins, g[f"s{s}_bins"][qi][:n])
            np.testing.assert_array_equal(oid, g[f"s{s}_ids"][qi][:n])
            np.testing.assert_array_equal(qt, g[f"s{s}_qtables"][qi])
            assert (qmin, qmax) == tuple(g[f"s{s}_qminmax"][qi])


def test_quick_adc_permuted_ids(golden):
    g = golden("quick_adc.npz")
    n2 = g["p_ids"].shape[0]
    t = O.compute_tables(g["codebooks"], g["queries"][0])
    bins, oid, qt, qmin, qmax = O.qadc_scan(g["codes"][:n2], g["p_ids"], t, 200, 64)
    np.testing.assert_array_equal(bins, g["p_bins"])
    np.testing.assert_array_equal(oid, g["p_out_ids"])
    np.testing.assert_array_equal(qt, g["p_qtables"])


def test_transpose_layout(golden):
    g = golden("quick_adc.npz")
    blocks = O.transpose_blocks(g["codes"], 4)
    np.testing.assert_array_equal(blocks, g["blocks"])
    back = O.detranspose_blocks(blocks, g["codes"].shape[0], 16, 4)
    np.testing.assert_array_equal(back, g["codes"])


def test_quantize_known_answers(golden):
    g = golden("quantize.npz")
    for p, (a, b) in enumerate(g["params"]):
        np.testing.assert_array_equal(O.quantize(a, b, g["values"]), g["bins"][p])
    np.testing.assert_array_equal(O.quantized_distances(g["codes"], g["qtables"]), g["qdist"])
    for bi, blk in enumerate(g["blocks"]):
        np.testing.assert_array_equal(O.qadc_block(blk, g["qtables"]), g["qblock"][bi])
    # test_fastscan.py:67-79 boundaries
    assert int(O.quantize(0.0, 8.0, 7.9999)) == 126
    assert int(O.quantize(0.0, 8.0, 8.0)) == 127


def _lists(g):
    sizes = g["list_sizes"]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    codes = [g["list_codes"][offs[c]:offs[c + 1]] for c in range(len(sizes))]
    ids = [g["list_ids"][offs[c]:offs[c + 1]] for c in range(len(sizes))]
    return codes, ids


def test_ivf_probes(golden):
    g = golden("ivf.npz")
    cells, dist = O.nearest_k(g["queries"].astype(np.float64), g["coarse"].astype(np.float64), 8)
    np.testing.assert_array_equal(cells, g["probe_cells"])
    np.testing.assert_array_equal(dist, g["probe_dist"])


@pytest.mark.parametrize("ma,r", [(1, 20), (4, 50), (16, 100), (32, 10)])
def test_ivf_query(golden, ma, r):
    g = golden("ivf.npz")
    codes, ids = _lists(g)
    for qi, q in enumerate(g["queries"]):
        d, i = O.query_ivf(g["coarse"], g["codebooks"], codes, ids, q, ma, r)
        n = len(d)
        np.testing.assert_array_equal(d, g[f"ma{ma}_r{r}_dist"][qi][:n])
        np.testing.assert_array_equal(i, g[f"ma{ma}_r{r}_ids"][qi][:n])
        assert np.all(g[f"ma{ma}_r{r}_ids"][qi][n:] == -1)


@pytest.mark.parametrize("tag", ["c1", "c3", "c2"])
def test_encode_golden(golden, tag):
    g = golden("encode.npz")
    books, x = g[f"{tag}_codebooks"], g[f"{tag}_x"]
    np.testing.assert_array_equal(O.encode(books, x), g[f"{tag}_codes"])
    np.testing.assert_array_equal(O.encode(books, x, g[f"{tag}_coarse"], g[f"{tag}_cells"]),
                                  g[f"{tag}_rescodes"])
    assert (g[f"{tag}_codes"][:50] == 0).all()  # tied duplicate centroid -> lowest index


QADC_IVF = [("built", 1, 20, 200), ("built", 4, 50, 30), ("built", 8, 100, 200), ("built", 24, 10, 5000),
            ("ties", 6, 100, 200), ("ties", 3, 40, 1), ("ties", 2, 250, 64)]


def qadc_ivf_lists(g, tag):
    sizes = g[f"{tag}_list_sizes"]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    codes = [g[f"{tag}_list_codes"][offs[c]:offs[c + 1]] for c in range(len(sizes))]
    ids = [g[f"{tag}_list_ids"][offs[c]:offs[c + 1]] for c in range(len(sizes))]
    return codes, ids


@pytest.mark.parametrize("tag,ma,r,ic", QADC_IVF)
def test_ivf_quick_adc_query(golden, tag, ma, r, ic):
    """query_ivf kernel='quick-adc' (ivf.py:185-190) vs the reference's outputs."""
    g = golden("ivf_qadc.npz")
    codes, ids = qadc_ivf_lists(g, tag)
    key = f"{tag}_ma{ma}_r{r}_i{ic}"
    for qi, q in enumerate(g["queries"]):
        d, i = O.query_ivf(g[f"{tag}_coarse"], g[f"{tag}_codebooks"], codes, ids, q, ma, r,
                           kernel="quick-adc", init_count=ic)
        n = len(d)
        np.testing.assert_array_equal(d, g[f"{key}_dist"][qi][:n])
        np.testing.assert_array_equal(i, g[f"{key}_ids"][qi][:n])
        assert np.all(g[f"{key}_ids"][qi][n:] == -1)


def _split(sizes, codes, ids):
    offs = np.concatenate([[0], np.cumsum(sizes)])
    return ([codes[offs[c]:offs[c + 1]] for c in range(len(sizes))],
            [ids[offs[c]:offs[c + 1]] for c in range(len(sizes))])


def test_fp64_queries(golden):
    """float64 queries float32 cannot represent: the reference computes from
    float64(query) (quantizer.py:85-89, ivf.py:170) -- the oracle too."""
    g = golden("fp64.npz")
    qs = g["queries"]
    assert qs.dtype == np.float64
    ids = np.arange(g["codes8"].shape[0])
    lc, li = _split(g["list_sizes"], g["list_codes"], g["list_ids"])
    lc4, li4 = _split(g["list4_sizes"], g["list4_codes"], g["list4_ids"])
    for qi, q in enumerate(qs):
        t = O.compute_tables(g["pq8_books"], q)
        np.testing.assert_array_equal(t.view(np.uint32), g["tables8"][qi].view(np.uint32))
        d, i = O.scan(g["codes8"], ids, t, 20)
        np.testing.assert_array_equal(d, g["scan_dist"][qi])
        np.testing.assert_array_equal(i, g["scan_ids"][qi])
        b, i, _, _, _ = O.qadc_scan(g["codes4"], ids, O.compute_tables(g["pq4_books"], q), 200, 30)
        np.testing.assert_array_equal(b, g["qadc_bins"][qi])
        np.testing.assert_array_equal(i, g["qadc_ids"][qi])
        d, i = O.query_ivf(g["coarse"], g["ivf_books"], lc, li, q, 5, 25)
        np.testing.assert_array_equal(d, g["ivf_dist"][qi])
        np.testing.assert_array_equal(i, g["ivf_ids"][qi])
        d, i = O.query_ivf(g["coarse4"], g["ivf4_books"], lc4, li4, q, 3, 15, kernel="quick-adc", init_count=50)
        np.testing.assert_array_equal(d, g["ivfq_dist"][qi])
        np.testing.assert_array_equal(i, g["ivfq_ids"][qi])
    cells, dist = O.nearest_k(qs, g["coarse"].astype(np.float64), 7)
    np.testing.assert_array_equal(cells, g["probe_cells"])
    np.testing.assert_array_equal(dist, g["probe_dist"])
    np.testing.assert_array_equal(O.encode(g["pq8_books"], g["enc_x"]), g["enc_codes"])
