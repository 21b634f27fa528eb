"""GPU: Quick ADC at large n -- the prefix-sample threshold (strict bin
threshold after the prefix when ids increase in storage order), tcgen05
launches chunked over tile ranges, bin-0 saturation (THETA_NONE), heavy ties
and explicit ids -- all bit-exact against the oracle."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from tests.helpers import kmeans_books, mixture

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def big():
    rng = np.random.default_rng(31)
    x = mixture(rng, 30_000, 64, comps=64)
    books = kmeans_books(x[:20_000], 16, 16, iters=3)
    n = 6_000_000
    codes = rng.integers(0, 16, (n, 16), dtype=np.uint8)
    qs = mixture(np.random.default_rng(32), 300, 64, comps=64)
    return books, codes, qs


def _run(books, codes, qs, r, init, ids=None, opts=None):
    ctx = P.Context(0)
    for k, v in (opts or {}).items():
        ctx.set_option(k, v)
    pq = P.ProductQuantizer(16, 4, 64, books)
    db = P.DeviceCodes(codes, 4, ids=ids, ctx=ctx)
    out = db.qadc_search(P.DeviceQuantizer(pq, ctx), qs, init, r)[:3]
    return out, ctx


def _check_oracle(books, codes, qs, out, r, init, qis, ids=None):
    bins, oids, cnt = out
    all_ids = np.arange(codes.shape[0], dtype=np.int64) if ids is None else ids
    for qi in qis:
        ob, oi, _, _, _ = O.qadc_scan(codes, all_ids, O.compute_tables(books, qs[qi]), init, r)
        assert cnt[qi] == len(ob)
        np.testing.assert_array_equal(bins[qi, :cnt[qi]], ob.astype(np.uint8))
        np.testing.assert_array_equal(oids[qi, :cnt[qi]], oi)


def test_large_auto_vs_oracle(big):
    books, codes, qs = big
    out, ctx = _run(books, codes, qs, 100, 1000)
    assert ctx.stat(P._lib.STAT_LAST_OVERFLOW) == 0
    _check_oracle(books, codes, qs, out, 100, 1000, (0, 150, 299))
    prmt, _ = _run(books, codes, qs, 100, 1000, opts={P._lib.OPT_SCAN4_ENGINE: 1})
    for a, b in zip(out, prmt):
        np.testing.assert_array_equal(a, b)


def test_tc_chunked_launches(big):
    books, codes, qs = big
    a, ca = _run(books, codes[:2_000_000], qs, 100, 1000, opts={P._lib.OPT_SCAN4_ENGINE: 2})
    b, cb = _run(books, codes[:2_000_000], qs, 100, 1000,
                 opts={P._lib.OPT_SCAN4_ENGINE: 2, P._lib.OPT_TC_CHUNK_TILES: 777})
    assert ca.stat(P._lib.STAT_LAST_SCAN_ENGINE) == 2 and cb.stat(P._lib.STAT_LAST_SCAN_ENGINE) == 2
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)


@pytest.mark.parametrize("engine", [1, 2])
def test_bin_zero_ties(big, engine):
    """Half the list is one code whose bin is 0 for the query (query = its
    reconstruction): theta = 0, the strict main threshold admits nothing and
    the answer is the r lowest ids of the prefix copies."""
    books, codes, qs = big
    rng = np.random.default_rng(33)
    n = 400_000
    c = codes[:n].copy()
    star = c[7].copy()
    c[rng.random(n) < 0.5] = star
    q = np.concatenate([books[j, star[j]] for j in range(16)])[None].astype(np.float32)
    qq = np.concatenate([q, qs[:5]])
    out, ctx = _run(books, c, qq, 100, 200, opts={P._lib.OPT_SCAN4_ENGINE: engine})
    assert out[0][0].max() == 0
    _check_oracle(books, c, qq, out, 100, 200, range(6))
    # explicit (permuted) ids: ties are broken by id, no strict threshold
    ids = rng.permutation(3 * n)[:n].astype(np.int64)
    out, _ = _run(books, c, qq, 100, 200, ids=ids, opts={P._lib.OPT_SCAN4_ENGINE: engine})
    _check_oracle(books, c, qq, out, 100, 200, range(6), ids=ids)


@pytest.mark.parametrize("engine", [1, 2])
@pytest.mark.parametrize("n,cap", [(20_000, 32768), (300_000, 60_000)])
def test_saturated_bins(big, engine, n, cap):
    """init_count 1 with queries next to the first code's reconstruction puts
    qmax just above qmin: nearly every sum saturates (bin 127 = min(S, 127)
    for any S >= 127), so the top-r is decided by a 127-bin tie broken by id
    -- codes with S > 127 must compete with S == 127 (theta 127 admits all)."""
    books, codes, qs = big
    c0 = codes[0]
    rec = np.concatenate([books[j, c0[j]] for j in range(16)]).astype(np.float32)
    rng = np.random.default_rng(34)
    qq = (rec[None] + rng.normal(0, 0.5, (12, 64))).astype(np.float32)
    out, ctx = _run(books, codes[:n], qq, 500, 1,
                    opts={P._lib.OPT_SCAN4_ENGINE: engine, P._lib.OPT_CAND_CAP: cap})
    assert (out[0][:, -1] == 127).all()
    _check_oracle(books, codes[:n], qq, out, 500, 1, range(12))
