"""GPU parity at BASELINE sizes (N = 1,000,000 codes, Q = 1,000): the whole
batch runs on the device; a seeded sample of queries is checked against the
CPU oracle (~50-90 ms per query per core), plus size-independent properties."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from paper_1712_02912_b200 import datagen as G

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def cfg1():
    return G.make_exhaustive("cfg1")


@pytest.fixture(scope="module")
def cfg0():
    return G.make_exhaustive("cfg0")


def test_cfg1_quick_adc_fullsize(cfg1):
    books, codes, qs = cfg1
    pq = P.ProductQuantizer(16, 4, 128, books)
    ctx = P.default_context()
    db = P.DeviceCodes(codes, 4)
    bins, ids, cnt, qt, qmm = db.qadc_search(P.DeviceQuantizer(pq), qs, 200, 100, want_tables=True)
    assert ctx.stat(3) == 0 and np.all(cnt == 100)
    all_ids = np.arange(codes.shape[0], dtype=np.int64)
    for qi in np.random.default_rng(0).choice(qs.shape[0], 6, replace=False):
        ob, oi, oqt, qmin, qmax = O.qadc_scan(codes, all_ids, O.compute_tables(books, qs[qi]), 200, 100)
        np.testing.assert_array_equal(bins[qi], ob.astype(np.uint8))
        np.testing.assert_array_equal(ids[qi], oi)
        np.testing.assert_array_equal(qt[qi], oqt)
        assert (qmm[qi, 0], qmm[qi, 1]) == (qmin, qmax)
    # property: every returned bin is the saturated quantized ADC of that code
    dense = db.quantized_distances(qt[:4])
    for qi in range(4):
        np.testing.assert_array_equal(dense[qi, ids[qi]], bins[qi])
        assert np.sum(dense[qi] < bins[qi, -1]) <= 100


def test_cfg1_sharded_equals_unsharded(cfg1):
    """Size-independent: 4 shards with the global prefix, merged == unsharded."""
    books, codes, qs = cfg1
    pq = P.ProductQuantizer(16, 4, 128, books)
    dq = P.DeviceQuantizer(pq)
    full = P.DeviceCodes(codes, 4).qadc_search(dq, qs, 200, 100)
    bounds = np.linspace(0, codes.shape[0], 5).astype(int)
    parts = []
    for g in range(4):
        sh = P.DeviceCodes(codes[bounds[g]:bounds[g + 1]], 4, id_base=int(bounds[g]))
        sh.set_prefix(codes[:200])
        parts.append(sh.qadc_search(dq, qs, 200, 100))
    d = np.stack([p[0].astype(np.float64) for p in parts])
    md, mi, mc = P.merge_topr(d, np.stack([p[1] for p in parts]), np.stack([p[2] for p in parts]), 100)
    np.testing.assert_array_equal(mi, full[1])
    np.testing.assert_array_equal(md.astype(np.uint8), full[0])


def test_cfg0_float_adc_fullsize(cfg0):
    books, codes, qs = cfg0
    pq = P.ProductQuantizer(8, 8, 128, books)
    ctx = P.default_context()
    d, i, c = P.DeviceCodes(codes, 8).adc_search(P.DeviceQuantizer(pq), qs, 100)
    assert ctx.stat(3) == 0 and np.all(c == 100)
    all_ids = np.arange(codes.shape[0], dtype=np.int64)
    for qi in np.random.default_rng(1).choice(qs.shape[0], 6, replace=False):
        od, oi = O.scan(codes, all_ids, O.compute_tables(books, qs[qi]), 100)
        np.testing.assert_array_equal(d[qi], od)
        np.testing.assert_array_equal(i[qi], oi)
    # drop-in single-query API == batched
    cl = P.CodeList(codes)
    got = P.scan(cl, P.compute_tables(pq, qs[3]), 100).items()
    assert got == list(zip(d[3].tolist(), i[3].tolist()))
