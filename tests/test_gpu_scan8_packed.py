"""Float ADC filter engines (scan8.cu): the packed two-queries-per-word kernel
(K3p, engine 5) against the oracle and against the u16 lane=query kernel
(engine 3) on shapes that exercise every layout corner: odd and non-multiple-
of-4 component counts (zero padding sub-slots), k < 256 (partial 64 KB slots),
m <= 8 (resident tables) and m > 8 (streamed quads), query counts that are not
a multiple of 32 (invalid halves of a packed word), a tail tile, and m > 64
(falls back to the u16 kernel).  Reference: scan (scan.py:197-203)."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from paper_1712_02912_b200 import _lib
from oracle import pqscan_oracle as O

pytestmark = pytest.mark.gpu


def _case(m, k, n, nq, seed, dsub=4, spread=1.0):
    rng = np.random.default_rng(seed)
    d = m * dsub
    books = (rng.normal(0, 1, (m, k, dsub)) * spread).astype(np.float32)
    codes = rng.integers(0, k, (n, m)).astype(np.uint8)
    # queries near reconstructed database rows so the top-r is well separated from the bulk
    rows = rng.integers(0, n, nq)
    base = np.stack([np.concatenate([books[j, codes[i, j]] for j in range(m)]) for i in rows])
    qs = (base + rng.normal(0, 0.3, base.shape)).astype(np.float32)
    return books, codes, qs


def _search(books, codes, qs, r, engine, b=8):
    m, k, dsub = books.shape
    ctx = P.Context(0)
    ctx.set_option(_lib.OPT_SCAN8_ENGINE, engine)
    full = np.zeros((m, 1 << b, dsub), np.float32)
    full[:, :k] = books
    if k < (1 << b):  # unused centroids far away (never the nearest); codes stay < k
        full[:, k:] = 1e3
    pq = P.ProductQuantizer(m, b, m * dsub, full)
    db = P.DeviceCodes(codes, 8, ctx=ctx)
    d, i, c = db.adc_search(P.DeviceQuantizer(pq, ctx), qs, r)
    return d, i, c, ctx, full


@pytest.mark.parametrize("m,k,n,nq", [
    (8, 256, 70_000, 37),     # resident, two quads, odd query count, tail tile
    (1, 256, 40_000, 5),      # one component (half of a pair)
    (3, 256, 40_000, 33),     # odd m: padded sub-slot in the second pair
    (5, 256, 40_000, 20),     # second quad holds one component
    (6, 256, 40_000, 64),
    (12, 256, 40_000, 40),    # streamed quads (m > 8)
    (18, 256, 36_000, 17),    # streamed, last quad holds two components
    (64, 256, 34_000, 9),     # cfg2 shape family, clip = 511
])
def test_packed_matches_oracle_and_u16(m, k, n, nq):
    books, codes, qs = _case(m, k, n, nq, seed=100 + m)
    r = 50
    d2, i2, c2, ctx2, full = _search(books, codes, qs, r, engine=2)
    assert ctx2.stat(_lib.STAT_LAST_SCAN_ENGINE) == 5
    assert ctx2.stat(_lib.STAT_LAST_OVERFLOW) == 0
    d1, i1, c1, ctx1, _ = _search(books, codes, qs, r, engine=1)
    assert ctx1.stat(_lib.STAT_LAST_SCAN_ENGINE) == 3
    np.testing.assert_array_equal(c1, c2)
    np.testing.assert_array_equal(d1, d2)
    np.testing.assert_array_equal(i1, i2)
    ids = np.arange(n, dtype=np.int64)
    for qi in range(0, nq, max(1, nq // 6)):
        od, oi = O.scan(codes, ids, O.compute_tables(full, qs[qi]), r)
        assert c2[qi] == len(od)
        np.testing.assert_array_equal(d2[qi, :c2[qi]], od)
        np.testing.assert_array_equal(i2[qi, :c2[qi]], oi)


def test_packed_small_k():
    """k = 100 < 256 entries: only the first k rows of a 64 KB slot are loaded."""
    m, k, n, nq = 8, 100, 40_000, 21
    rng = np.random.default_rng(5)
    books = rng.normal(0, 1, (m, k, 4)).astype(np.float32)
    codes = rng.integers(0, k, (n, m)).astype(np.uint8)
    qs = rng.normal(0, 1, (nq, m * 4)).astype(np.float32)
    ctx = P.Context(0)
    ctx.set_option(_lib.OPT_SCAN8_ENGINE, 2)
    # a quantizer with k = 128 (b = 7) whose upper 28 centroids are never used
    full = np.concatenate([books, np.full((m, 28, 4), 50.0, np.float32)], axis=1)
    pq = P.ProductQuantizer(m, 7, m * 4, full)
    db = P.DeviceCodes(codes, 8, ctx=ctx)
    d, i, c = db.adc_search(P.DeviceQuantizer(pq, ctx), qs, 30)
    assert ctx.stat(_lib.STAT_LAST_SCAN_ENGINE) == 5
    ids = np.arange(n, dtype=np.int64)
    for qi in range(0, nq, 4):
        od, oi = O.scan(codes, ids, O.compute_tables(full, qs[qi]), 30)
        np.testing.assert_array_equal(d[qi, :c[qi]], od)
        np.testing.assert_array_equal(i[qi, :c[qi]], oi)


def test_wide_m_uses_u16_engine():
    m, k, n, nq = 72, 256, 33_000, 6
    books, codes, qs = _case(m, k, n, nq, seed=9, dsub=2)
    d, i, c, ctx, full = _search(books, codes, qs, 20, engine=0)
    assert ctx.stat(_lib.STAT_LAST_SCAN_ENGINE) == 3
    ids = np.arange(n, dtype=np.int64)
    for qi in range(nq):
        od, oi = O.scan(codes, ids, O.compute_tables(full, qs[qi]), 20)
        np.testing.assert_array_equal(d[qi, :c[qi]], od)
        np.testing.assert_array_equal(i[qi, :c[qi]], oi)


def test_packed_heavy_ties_and_clipped_entries():
    """Identical codes (ties at the threshold) and a table with entries far above
    the clip value: clipped entries stay lower bounds, ties are all kept."""
    m, k, n, nq = 8, 256, 50_000, 8
    rng = np.random.default_rng(11)
    books = rng.normal(0, 1, (m, k, 4)).astype(np.float32)
    books[:, 200:] *= 400.0   # huge distances: saturate the 15-bit entries
    codes = rng.integers(0, 8, (n, m)).astype(np.uint8)   # 8^8 combos, many repeats of near ones
    codes[rng.integers(0, n, 5000)] = codes[0]
    codes[n // 2:, 3] = rng.integers(200, 256, n - n // 2).astype(np.uint8)
    qs = np.stack([np.concatenate([books[j, codes[0, j]] for j in range(m)])] * nq).astype(np.float32)
    qs += rng.normal(0, 0.05, qs.shape).astype(np.float32)
    d, i, c, ctx, full = _search(books, codes, qs, 100, engine=2)
    assert ctx.stat(_lib.STAT_LAST_SCAN_ENGINE) == 5
    ids = np.arange(n, dtype=np.int64)
    for qi in range(nq):
        od, oi = O.scan(codes, ids, O.compute_tables(full, qs[qi]), 100)
        np.testing.assert_array_equal(d[qi, :c[qi]], od)
        np.testing.assert_array_equal(i[qi, :c[qi]], oi)
