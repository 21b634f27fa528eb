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
