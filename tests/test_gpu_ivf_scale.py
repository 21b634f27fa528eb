"""GPU: IVFADC on an index built on the device (datagen.make_ivf_device:
coarse k-means, assignment, exact residual encode, lists in cell order) at
a mid size (N = 2M, K = 4096, nprobe 64) -- search results bit-exact against
the oracle's query_ivf over the same lists."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def index():
    from paper_1712_02912_b200 import datagen as G

    ctx = P.default_context()
    books, coarse, sizes, codes, ids, queries = G.make_ivf_device(
        "cfg3", lambda b: P.DeviceQuantizer(P.ProductQuantizer(8, 8, 128, b), ctx), n=2_000_000, K=4096, nq=300,
        coarse_iters=4)
    return books, coarse, sizes, codes, ids, queries


def test_device_index_is_consistent(index):
    books, coarse, sizes, codes, ids, queries = index
    assert int(sizes.sum()) == codes.shape[0] == ids.shape[0]
    idh = ids.cpu().numpy()
    assert np.array_equal(np.sort(idh), np.arange(idh.shape[0]))
    offs = np.concatenate([[0], np.cumsum(sizes)])
    for c in (0, 17, 4095):  # ids ascending inside a list (build_ivf's flatnonzero order)
        assert np.all(np.diff(idh[offs[c]:offs[c + 1]]) > 0)


def test_ivf_search_vs_oracle(index):
    books, coarse, sizes, codes, ids, queries = index
    pq = P.ProductQuantizer(8, 8, 128, books)
    ivf = P.DeviceIvf.from_arrays(pq, coarse, sizes, codes, ids)
    d, i, c = ivf.search(queries, 64, 100)
    ch, cb, ih = coarse.cpu().numpy(), codes.cpu().numpy(), ids.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(sizes)])
    lc = [cb[offs[k]:offs[k + 1]] for k in range(len(sizes))]
    li = [ih[offs[k]:offs[k + 1]] for k in range(len(sizes))]
    for qi in (0, 123, 299):
        od, oi = O.query_ivf(ch, books, lc, li, queries[qi], 64, 100)
        assert c[qi] == len(od)
        np.testing.assert_array_equal(d[qi, :c[qi]], od)
        np.testing.assert_array_equal(i[qi, :c[qi]], oi)


def test_probe_sets_exact_many_queries(index):
    """K7 probes (TF32 GEMM + certified fp64 re-score) == nearest_k
    (_dist.py:42-67) for all 300 queries: same cells, same order, same fp64
    distances -- incl. the cfg3 geometry (queries inside a mixture component
    tiled by many centroids)."""
    books, coarse, sizes, codes, ids, queries = index
    pq = P.ProductQuantizer(8, 8, 128, books)
    ivf = P.DeviceIvf.from_arrays(pq, coarse, sizes, codes, ids)
    for ma in (1, 64, 300):
        cells, dist = ivf.probe(queries, ma)
        oc, od = O.nearest_k(queries.astype(np.float64), coarse.cpu().numpy().astype(np.float64), ma)
        np.testing.assert_array_equal(cells, oc)
        np.testing.assert_array_equal(dist, od)


def test_packed_list_scan_matches_float_list_scan_and_oracle(index):
    """The packed integer pre-filter (K8p, engine 6) keeps a superset of the
    fp32 filter's survivors, so after the refine step both engines hand the
    same candidates to the exact rerank: identical results for every query,
    float32 and float64 queries, several (ma, r), and == oracle on a sample."""
    from paper_1712_02912_b200 import _lib

    books, coarse, sizes, codes, ids, queries = index
    pq = P.ProductQuantizer(8, 8, 128, books)
    res = {}
    for eng in (1, 2):
        ctx = P.Context(0)
        ctx.set_option(_lib.OPT_IVF_ENGINE, eng)
        ivf = P.DeviceIvf.from_arrays(pq, coarse, sizes, codes, ids, ctx=ctx)
        out = []
        for qs, ma, r in ((queries, 64, 100), (queries[:50].astype(np.float64) + 1e-9, 8, 10), (queries[:33], 200, 500)):
            d, i, c = ivf.search(qs, ma, r)
            assert ctx.stat(_lib.STAT_LAST_SCAN_ENGINE) == (4 if eng == 1 else 6)
            assert ctx.stat(_lib.STAT_LAST_OVERFLOW) == 0
            out.append((d.copy(), i.copy(), c.copy()))
        res[eng] = out
    for (d1, i1, c1), (d2, i2, c2) in zip(res[1], res[2]):
        np.testing.assert_array_equal(c1, c2)
        np.testing.assert_array_equal(d1, d2)
        np.testing.assert_array_equal(i1, i2)
    ch, cb, ih = coarse.cpu().numpy(), codes.cpu().numpy(), ids.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(sizes)])
    lc = [cb[offs[k]:offs[k + 1]] for k in range(len(sizes))]
    li = [ih[offs[k]:offs[k + 1]] for k in range(len(sizes))]
    d, i, c = res[2][0]
    for qi in (1, 77, 150, 298):
        od, oi = O.query_ivf(ch, books, lc, li, queries[qi], 64, 100)
        np.testing.assert_array_equal(d[qi, :c[qi]], od)
        np.testing.assert_array_equal(i[qi, :c[qi]], oi)


def test_packed_list_scan_small_index_all_kept():
    """Tiny lists: the threshold sample holds fewer than r codes (theta = +inf),
    so the packed scan keeps every probed code (scale 0) -- and a record
    overflow falls back to the float list scan; results == oracle either way."""
    from paper_1712_02912_b200 import _lib

    rng = np.random.default_rng(12)
    d, K, n = 32, 16, 3000
    x = rng.normal(0, 4, (n, d)).astype(np.float32)
    coarse = x[:K].copy()
    assign = ((x[:, None, :] - coarse[None]) ** 2).sum(-1).argmin(1)
    books = rng.normal(0, 2, (8, 256, 4)).astype(np.float32)
    codes = rng.integers(0, 256, (n, 8)).astype(np.uint8)
    lists_c = [codes[assign == c] for c in range(K)]
    lists_i = [np.flatnonzero(assign == c).astype(np.int64) for c in range(K)]
    pq = P.ProductQuantizer(8, 8, d, books)
    ctx = P.Context(0)
    ctx.set_option(_lib.OPT_IVF_ENGINE, 2)
    idx = P.IvfIndex(coarse, pq, [P.CodeList(a, b) for a, b in zip(lists_c, lists_i)])
    ivf = P.DeviceIvf(idx, ctx=ctx)
    qs = (x[:20] + 0.5).astype(np.float32)
    dd, ii, cc = ivf.search(qs, 5, 400)
    for qi in range(0, 20, 3):
        od, oi = O.query_ivf(coarse, books, lists_c, lists_i, qs[qi], 5, 400)
        assert cc[qi] == len(od)
        np.testing.assert_array_equal(dd[qi, :cc[qi]], od)
        np.testing.assert_array_equal(ii[qi, :cc[qi]], oi)


def test_packed_list_scan_long_lists_many_passes():
    """Few, long lists probed by many queries: every list spans several staged
    code chunks (> 3072 codes) and takes many 8-query passes (double-buffered
    table halves, raw-table prefetch across passes and lists); packed engine ==
    float engine for all queries and == oracle on a sample."""
    from paper_1712_02912_b200 import _lib

    rng = np.random.default_rng(21)
    d, K, n, nq = 32, 12, 150_000, 200
    centers = rng.uniform(0, 100, (K, d)).astype(np.float32)
    lab = rng.integers(0, K, n)
    x = (centers[lab] + rng.normal(0, 6, (n, d))).astype(np.float32)
    coarse = centers + rng.normal(0, 1, (K, d)).astype(np.float32)
    assign, _ = P.nearest(x, coarse)
    books = rng.normal(0, 5, (8, 256, 4)).astype(np.float32)
    pq = P.ProductQuantizer(8, 8, d, books)
    res = (x.astype(np.float64) - coarse[assign].astype(np.float64)).astype(np.float32)
    codes = P.DeviceQuantizer(pq).encode(res)
    codes = np.asarray(codes)
    lists_c = [codes[assign == c] for c in range(K)]
    lists_i = [np.flatnonzero(assign == c).astype(np.int64) for c in range(K)]
    assert max(len(l) for l in lists_c) > 2 * 3072
    qs = (x[rng.integers(0, n, nq)] + rng.normal(0, 2, (nq, d))).astype(np.float32)
    idx = P.IvfIndex(coarse, pq, [P.CodeList(a, b) for a, b in zip(lists_c, lists_i)])
    out = {}
    for eng in (1, 2):
        ctx = P.Context(0)
        ctx.set_option(_lib.OPT_IVF_ENGINE, eng)
        ivf = P.DeviceIvf(idx, ctx=ctx)
        out[eng] = ivf.search(qs, 4, 100)
        assert ctx.stat(_lib.STAT_LAST_SCAN_ENGINE) == (4 if eng == 1 else 6)
        assert ctx.stat(_lib.STAT_LAST_OVERFLOW) == 0
    for a, b in zip(out[1], out[2]):
        np.testing.assert_array_equal(a, b)
    dd, ii, cc = out[2]
    for qi in range(0, nq, 37):
        od, oi = O.query_ivf(coarse, books, lists_c, lists_i, qs[qi], 4, 100)
        assert cc[qi] == len(od)
        np.testing.assert_array_equal(dd[qi, :cc[qi]], od)
        np.testing.assert_array_equal(ii[qi, :cc[qi]], oi)
