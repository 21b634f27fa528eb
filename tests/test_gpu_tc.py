"""GPU: the tcgen05 (kind::i8 one-hot GEMM) Quick ADC scan and the PRMT scan
give identical results, and both match the oracle."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from tests.helpers import encode, kmeans_books, mixture

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def data():
    rng = np.random.default_rng(21)
    x = mixture(rng, 300_000, 64, comps=128)
    books = kmeans_books(x[:20000], 16, 16, iters=4)
    codes = encode(books, x)
    qs = mixture(np.random.default_rng(22), 300, 64, comps=128)  # 2 query groups of 256 (one partial)
    return books, codes, qs


def _search(books, codes, qs, engine, r=100, init=200):
    ctx = P.Context(0)
    ctx.set_option(4, engine)
    pq = P.ProductQuantizer(16, 4, 64, books)
    db = P.DeviceCodes(codes, 4, ctx=ctx)
    out = db.qadc_search(P.DeviceQuantizer(pq, ctx), qs, init, r, want_tables=True)
    assert ctx.stat(3) == 0
    return out


def test_tc_equals_prmt(data):
    books, codes, qs = data
    tc = _search(books, codes, qs, 2)
    pr = _search(books, codes, qs, 1)
    for a, b in zip(tc, pr):
        np.testing.assert_array_equal(a, b)


def test_tc_vs_oracle(data):
    books, codes, qs = data
    bins, ids, cnt, qt, qmm = _search(books, codes, qs, 2, r=50, init=1000)
    all_ids = np.arange(codes.shape[0], dtype=np.int64)
    for qi in (0, 131, 257, 299):
        ob, oi, oqt, qmin, qmax = O.qadc_scan(codes, all_ids, O.compute_tables(books, qs[qi]), 1000, 50)
        np.testing.assert_array_equal(bins[qi, :cnt[qi]], ob.astype(np.uint8))
        np.testing.assert_array_equal(ids[qi, :cnt[qi]], oi)


def test_tc_odd_sizes(data):
    """n not a multiple of the 128-code tile, few queries (partial group)."""
    books, codes, qs = data
    n = 99_999
    tc = _search(books, codes[:n], qs[:37], 2, r=20)
    pr = _search(books, codes[:n], qs[:37], 1, r=20)
    for a, b in zip(tc, pr):
        np.testing.assert_array_equal(a, b)


def test_graph_replay_matches_direct(data):
    """The Quick ADC device phase is captured as a CUDA graph on the second
    identical call and replayed afterwards: replays with new query batches of
    the same shape (and host/device io) equal the uncaptured result."""
    import torch

    books, codes, qs = data
    pq = P.ProductQuantizer(16, 4, 64, books)
    ctx = P.Context(0)
    db = P.DeviceCodes(codes, 4, ctx=ctx)
    dq = P.DeviceQuantizer(pq, ctx)
    rng = np.random.default_rng(9)
    batches = [qs + rng.normal(0, 3, qs.shape).astype(np.float32) for _ in range(4)]
    got = [db.qadc_search(dq, b, 200, 100, want_tables=True) for b in batches]       # run, capture, replay, replay
    got.append(db.qadc_search(dq, torch.from_numpy(batches[1]).cuda(), 200, 100, want_tables=True))
    ref_ctx = P.Context(0)
    ref_db = P.DeviceCodes(codes, 4, ctx=ref_ctx)
    ref_dq = P.DeviceQuantizer(pq, ref_ctx)
    for k, b in enumerate(batches + [batches[1]]):
        want = ref_db.qadc_search(ref_dq, b, 200, 100, want_tables=True)
        ref_db = P.DeviceCodes(codes, 4, ctx=ref_ctx)   # new handle: never replays
        for u, v in zip(got[k], want):
            u = u.cpu().numpy() if hasattr(u, "cpu") else u
            np.testing.assert_array_equal(u, v)
