"""GPU parity at the remaining BASELINE sizes: cfg2 (d=960, 64x8, N=1M),
cfg3 (IVFADC, N=1e8, K=65,536, nprobe 64) and one 125M-code shard of cfg4
(billion-scale Quick ADC), generated and indexed on the GPU.  A seeded sample
of queries is checked bit-exactly against the CPU oracle (cfg3: query_ivf over
a host copy of the whole index; cfg4: the oracle Quick ADC over all 125M
codes of the shard with the global prefix)."""

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


def test_cfg2_float_adc_fullsize():
    books, codes, qs = G.make_exhaustive("cfg2", nq=64)
    pq = P.ProductQuantizer(64, 8, 960, books)
    ctx = P.default_context()
    d, i, c = P.DeviceCodes(codes, 8).adc_search(P.DeviceQuantizer(pq), qs, 100)
    assert ctx.stat(3) == 0 and np.all(c == 100)
    all_ids = np.arange(codes.shape[0], dtype=np.int64)
    for qi in (0, 31, 63):
        od, oi = O.scan(codes, all_ids, O.compute_tables(books, qs[qi]), 100)
        np.testing.assert_array_equal(d[qi], od)
        np.testing.assert_array_equal(i[qi], oi)


def test_cfg3_ivfadc_fullsize():
    import torch

    ctx = P.default_context()
    books, coarse, sizes, codes, ids, qs = G.make_ivf_device(
        "cfg3", lambda b: P.DeviceQuantizer(P.ProductQuantizer(8, 8, 128, b), ctx), nq=2000)
    ivf = P.DeviceIvf.from_arrays(P.ProductQuantizer(8, 8, 128, books), coarse, sizes, codes, ids)
    d, i, c = ivf.search(torch.from_numpy(qs).cuda(), 64, 100)
    d, i, c = d.cpu().numpy(), i.cpu().numpy(), c.cpu().numpy()
    assert ctx.stat(3) == 0 and np.all(c == 100)
    ch, cb, ih = coarse.cpu().numpy(), codes.cpu().numpy(), ids.cpu().numpy()
    del codes, ids
    offs = np.concatenate([[0], np.cumsum(sizes)])
    lc = [cb[offs[k]:offs[k + 1]] for k in range(len(sizes))]
    li = [ih[offs[k]:offs[k + 1]] for k in range(len(sizes))]
    for qi in np.random.default_rng(3).choice(qs.shape[0], 4, replace=False):
        od, oi = O.query_ivf(ch, books, lc, li, qs[qi], 64, 100)
        np.testing.assert_array_equal(d[qi], od)
        np.testing.assert_array_equal(i[qi], oi)


def test_cfg4_shard_quick_adc_fullsize():
    ctx = P.default_context()
    rank, world = 3, 8   # a middle shard: ids 375M..500M, global prefix from shard 0
    books, codes, prefix, qs = G.make_quick_adc_shard(
        "cfg4", rank, world, lambda b: P.DeviceQuantizer(P.ProductQuantizer(16, 4, 96, b), ctx), nq=2000)
    n = codes.shape[0]
    db = P.DeviceCodes(codes, 4, id_base=rank * n)
    db.set_prefix(prefix)
    pq = P.ProductQuantizer(16, 4, 96, books)
    bins, ids, cnt, qt, qmm = db.qadc_search(P.DeviceQuantizer(pq), qs, 1000, 100, want_tables=True)
    assert ctx.stat(3) == 0 and np.all(cnt == 100)
    ch = codes.cpu().numpy()
    ph = prefix.cpu().numpy()
    del codes
    for qi in (0, 1234):
        t = O.compute_tables(books, qs[qi])
        qmin, qmax = O.qadc_params(t, ph, 1000, 100)          # global prefix (quickadc.py:129-137)
        assert (qmm[qi, 0], qmm[qi, 1]) == (qmin, qmax)
        qtab = O.quantize(qmin, qmax, t)
        np.testing.assert_array_equal(qt[qi], qtab)
        best_d, best_i = None, None
        for lo in range(0, n, 10_000_000):                    # chunked, memory-bounded
            hi = min(n, lo + 10_000_000)
            dist = O.quantized_distances(ch[lo:hi], qtab).astype(np.float64)
            cd, ci = O.select_best(dist, np.arange(lo, hi, dtype=np.int64) + rank * n, 100)
            if best_d is None:
                best_d, best_i = cd, ci
            else:
                best_d, best_i = O.select_best(np.concatenate([best_d, cd]), np.concatenate([best_i, ci]), 100)
        np.testing.assert_array_equal(bins[qi], best_d.astype(np.uint8))
        np.testing.assert_array_equal(ids[qi], best_i)
