"""GPU: derived-quantizer two-pass search (derived.cu) and query_ivf
kernel='derived' -- identical to the reference's outputs (golden) and to the
oracle at a larger size (both admission regimes: >= r2 codes below the
saturated bucket, and the d = 255 storage-order admission)."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from paper_1712_02912_b200 import derived as D
from tests.helpers import encode, kmeans_books, mixture
from tests.test_derived_host import IVF_SETTINGS, SETTINGS, ivf_lists

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _dpq(g, books="books", derived="derived", bbar=4):
    m, k, dsub = g[books].shape
    pq = P.ProductQuantizer(m, int(np.log2(k)), m * dsub, g[books])
    return D.DerivedPQ(pq, int(np.log2(g[derived].shape[1])), g[derived])


@pytest.mark.parametrize("r,r2", SETTINGS)
def test_two_pass_golden(golden, r, r2):
    g = golden("derived.npz")
    dpq = _dpq(g)
    db = P.CodeList(g["codes"], g["ids"])
    for qi, q in enumerate(g["queries"]):
        items = P.search_two_pass(dpq, db, q, r, r2).items()
        n = len(items)
        assert [d for d, _ in items] == g[f"r{r}_r2{r2}_dist"][qi][:n].tolist()
        assert [i for _, i in items] == g[f"r{r}_r2{r2}_ids"][qi][:n].tolist()
    d, i, c = D.search_two_pass_batch(dpq, db, g["queries"], r, r2)
    for qi in range(len(g["queries"])):
        n = int(c[qi])
        np.testing.assert_array_equal(d[qi, :n], g[f"r{r}_r2{r2}_dist"][qi][:n])
        np.testing.assert_array_equal(i[qi, :n], g[f"r{r}_r2{r2}_ids"][qi][:n])


@pytest.mark.parametrize("ma,r,r2", IVF_SETTINGS)
def test_ivf_derived_golden(golden, ma, r, r2):
    g = golden("derived.npz")
    dpq = _dpq(g, "ivf_books", "ivf_derived")
    codes, ids = ivf_lists(g)
    idx = P.IvfIndex(g["ivf_coarse"], dpq.pq, [P.CodeList(c, i) for c, i in zip(codes, ids)], dpq=dpq)
    for qi, q in enumerate(g["queries"]):
        items = P.query_ivf(idx, q, ma=ma, r=r, kernel="derived", r2=r2).items()
        n = len(items)
        assert [d for d, _ in items] == g[f"ivf_ma{ma}_r{r}_r2{r2}_dist"][qi][:n].tolist()
        assert [i for _, i in items] == g[f"ivf_ma{ma}_r{r}_r2{r2}_ids"][qi][:n].tolist()


def test_compact_tables_bitwise(golden):
    g = golden("derived.npz")
    dpq = _dpq(g)
    for q in g["queries"]:
        np.testing.assert_array_equal(P.compute_compact_tables(dpq, q).tables.view(np.uint32),
                                      O.compute_tables(g["derived"], q).view(np.uint32))


def test_two_pass_vs_oracle_large():
    """300k codes (m=8, b=8, bbar=4): r2 well below n (bucket bound) and above
    the count of unsaturated codes (storage-order admission of d = 255)."""
    rng = np.random.default_rng(9)
    x = mixture(rng, 300_000, 64, comps=64)
    books = kmeans_books(x[:20000], 8, 256, iters=3)
    derived = books.reshape(8, 16, 16, 8).mean(axis=1).astype(np.float32)   # any (m, 16, dsub) codebooks
    codes = encode(books, x)
    ids = rng.permutation(10**6)[:300_000].astype(np.int64)
    dpq = D.DerivedPQ(P.ProductQuantizer(8, 8, 64, books), 4, derived)
    db = P.CodeList(codes, ids)
    qs = x[rng.choice(300_000, 6, replace=False)] + rng.normal(0, 3, (6, 64)).astype(np.float32)
    for r, r2 in [(100, 9000), (10, 250_000), (1000, 20_000), (50, 400_000)]:
        d, i, c = D.search_two_pass_batch(dpq, db, qs, r, r2)
        for qi in (0, 3, 5):
            od, oi = O.search_two_pass(books, derived, codes, ids, qs[qi], r, r2)
            np.testing.assert_array_equal(d[qi, :int(c[qi])], od)
            np.testing.assert_array_equal(i[qi, :int(c[qi])], oi)
