"""GPU parity of query_ivf kernel='quick-adc' (ivf.py:185-190, device kernel
ivf_qadc.cu): the golden fixtures written by the reference (built index;
permuted ids with heavy bin ties, empty and tiny lists; init_count below r
and above every list) and the CPU oracle on a larger seeded index.  Bar:
bit-exact rescaled fp64 distances and ids."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from tests.helpers import kmeans_books, mixture
from tests.test_oracle_golden import QADC_IVF, qadc_ivf_lists

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _index(g, tag):
    books = g[f"{tag}_codebooks"]
    m, _, dsub = books.shape
    pq = P.ProductQuantizer(m, 4, m * dsub, books)
    codes, ids = qadc_ivf_lists(g, tag)
    return P.IvfIndex(g[f"{tag}_coarse"], pq, [P.CodeList(c, i) for c, i in zip(codes, ids)])


@pytest.mark.parametrize("tag,ma,r,ic", QADC_IVF)
def test_ivf_quick_adc_golden(golden, tag, ma, r, ic):
    g = golden("ivf_qadc.npz")
    idx = _index(g, tag)
    key = f"{tag}_ma{ma}_r{r}_i{ic}"
    for qi, q in enumerate(g["queries"]):
        items = P.query_ivf(idx, q, ma=ma, r=r, kernel="quick-adc", init_count=ic).items()
        n = len(items)
        assert [d for d, _ in items] == g[f"{key}_dist"][qi][:n].tolist()
        assert [i for _, i in items] == g[f"{key}_ids"][qi][:n].tolist()
        assert np.all(g[f"{key}_ids"][qi][n:] == -1)
    # batched form == per-query form
    d, i, c = P.ivf.query_ivf_batch(idx, g["queries"], ma, r, kernel="quick_adc", init_count=ic)
    for qi in range(len(g["queries"])):
        n = int(c[qi])
        np.testing.assert_array_equal(d[qi, :n], g[f"{key}_dist"][qi][:n])
        np.testing.assert_array_equal(i[qi, :n], g[f"{key}_ids"][qi][:n])


def test_ivf_quick_adc_errors(golden):
    g = golden("ivf_qadc.npz")
    idx = _index(g, "built")
    q = g["queries"][0]
    with pytest.raises(ValueError):
        P.query_ivf(idx, q, ma=2, r=10, kernel="quick-adc", init_count=0)
    with pytest.raises(ValueError):
        P.query_ivf(idx, q, ma=0, r=10, kernel="quick-adc")
    with pytest.raises(ValueError):
        P.query_ivf(idx, q, ma=2, r=0, kernel="quick-adc")


def test_ivf_quick_adc_vs_oracle():
    """16x4 residual codes, K=256 lists (~2.3k codes each), 64 queries, ma=16:
    larger lists than the fixtures, long tie runs at the cut bin."""
    rng = np.random.default_rng(21)
    d, K, n = 64, 256, 600_000
    x = mixture(rng, n, d, comps=128)
    coarse = x[rng.choice(n, K, replace=False)].copy()
    c64 = coarse.astype(np.float64)
    xc = np.empty(n, np.int64)
    for s in range(0, n, 4096):       # nearest coarse cell (data prep; ties irrelevant here)
        xs = x[s:s + 4096].astype(np.float64)
        xc[s:s + 4096] = ((xs * xs).sum(1)[:, None] - 2 * xs @ c64.T + (c64 * c64).sum(1)[None]).argmin(1)
    res = (x[:40000].astype(np.float64) - c64[xc[:40000]]).astype(np.float32)
    books = kmeans_books(res, 16, 16, iters=4)
    pq = P.ProductQuantizer(16, 4, d, books)
    dq = P.DeviceQuantizer(pq)
    codes = dq.encode(x, coarse=coarse, cells=xc)
    ids = rng.permutation(n).astype(np.int64)
    order = np.argsort(xc, kind="stable")
    sizes = np.bincount(xc, minlength=K).astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    lc = [codes[order[offs[c]:offs[c + 1]]] for c in range(K)]
    li = [ids[order[offs[c]:offs[c + 1]]] for c in range(K)]
    idx = P.IvfIndex(coarse, pq, [P.CodeList(a, b) for a, b in zip(lc, li)])
    qs = x[rng.choice(n, 64, replace=False)] + rng.normal(0, 4, (64, d)).astype(np.float32)
    dd, ii, cc = P.ivf.query_ivf_batch(idx, qs, 16, 100, kernel="quick-adc", init_count=200)
    assert np.all(cc == 100)
    for qi in (0, 17, 42, 63):
        od, oi = O.query_ivf(coarse, books, lc, li, qs[qi], 16, 100, kernel="quick-adc", init_count=200)
        np.testing.assert_array_equal(dd[qi], od)
        np.testing.assert_array_equal(ii[qi], oi)
