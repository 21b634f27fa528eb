"""GPU tests of the drop-in boundary: float64 queries end to end (the
reference computes from float64(query): quantizer.py:85-89, ivf.py:170,
encode quantizer.py:319-323), CUDA-graph replay after a code list is
destroyed and another of the same size created, and device-cache coherence
of the drop-in containers (in-place edits refused, rebinding re-uploads)."""

import gc

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


def _split(sizes, codes, ids):
    offs = np.concatenate([[0], np.cumsum(sizes)])
    return ([codes[offs[c]:offs[c + 1]] for c in range(len(sizes))],
            [ids[offs[c]:offs[c + 1]] for c in range(len(sizes))])


# ---------------------------------------------------------------- float64 queries
def test_fp64_golden(golden):
    """Reference outputs for float64 queries float32 cannot represent."""
    g = golden("fp64.npz")
    qs = g["queries"]
    pq8 = P.ProductQuantizer(4, 8, 32, g["pq8_books"])
    pq4 = P.ProductQuantizer(8, 4, 32, g["pq4_books"])
    cl = P.CodeList(g["codes8"])
    tl = P.transpose_blocks(P.CodeList(g["codes4"]), 4)
    lc, li = _split(g["list_sizes"], g["list_codes"], g["list_ids"])
    idx = P.IvfIndex(g["coarse"], P.ProductQuantizer(4, 8, 32, g["ivf_books"]),
                     [P.CodeList(c, i) for c, i in zip(lc, li)])
    lc4, li4 = _split(g["list4_sizes"], g["list4_codes"], g["list4_ids"])
    idx4 = P.IvfIndex(g["coarse4"], P.ProductQuantizer(8, 4, 32, g["ivf4_books"]),
                      [P.CodeList(c, i) for c, i in zip(lc4, li4)])
    for qi, q in enumerate(qs):
        t = P.compute_tables(pq8, q)
        np.testing.assert_array_equal(t.tables.view(np.uint32), g["tables8"][qi].view(np.uint32))
        assert P.scan(cl, t, 20).items() == list(zip(g["scan_dist"][qi].tolist(), g["scan_ids"][qi].tolist()))
        nset, _ = P.qadc_scan(tl, P.compute_tables(pq4, q), 200, 30)
        assert nset.items() == list(zip(g["qadc_bins"][qi].tolist(), g["qadc_ids"][qi].tolist()))
        got = P.query_ivf(idx, q, ma=5, r=25).items()
        assert got == list(zip(g["ivf_dist"][qi].tolist(), g["ivf_ids"][qi].tolist()))
        got = P.query_ivf(idx4, q, ma=3, r=15, kernel="quick-adc", init_count=50).items()
        assert got == list(zip(g["ivfq_dist"][qi].tolist(), g["ivfq_ids"][qi].tolist()))
    cells, dist = P.device_index(idx).probe(qs, 7)
    np.testing.assert_array_equal(cells, g["probe_cells"])
    np.testing.assert_array_equal(dist, g["probe_dist"])
    np.testing.assert_array_equal(P.encode(pq8, g["enc_x"]), g["enc_codes"])


def test_fp64_batched_host_and_device():
    """Batched APIs on float64 numpy arrays and float64 CUDA tensors ==
    the oracle computed from the float64 values (nothing rounded)."""
    import torch

    rng = np.random.default_rng(41)
    x = mixture(rng, 60_000, 64, comps=64)
    books8 = kmeans_books(x[:8000], 8, 256, iters=2)
    books4 = kmeans_books(x[:8000], 16, 16, iters=3)
    c8, c4 = encode(books8, x), encode(books4, x)
    qs = x[:12].astype(np.float64) + rng.normal(0, 3.0, (12, 64))
    ids = np.arange(len(x))
    dq8 = P.DeviceQuantizer(P.ProductQuantizer(8, 8, 64, books8))
    dq4 = P.DeviceQuantizer(P.ProductQuantizer(16, 4, 64, books4))
    db8, db4 = P.DeviceCodes(c8, 8), P.DeviceCodes(c4, 4)
    for arg in (qs, torch.from_numpy(qs).cuda()):
        d, i, c = db8.adc_search(dq8, arg, 50)
        b, bi, bc, _, _ = db4.qadc_search(dq4, arg, 200, 50)
        d, i, b, bi = (t.cpu().numpy() if hasattr(t, "cpu") else t for t in (d, i, b, bi))
        for qi, q in enumerate(qs):
            od, oi = O.scan(c8, ids, O.compute_tables(books8, q), 50)
            np.testing.assert_array_equal(d[qi], od)
            np.testing.assert_array_equal(i[qi], oi)
            ob, oi4, _, _, _ = O.qadc_scan(c4, ids, O.compute_tables(books4, q), 200, 50)
            np.testing.assert_array_equal(b[qi], ob)
            np.testing.assert_array_equal(bi[qi], oi4)
    # float32 input still goes through the float32 entry points, same answers
    t32 = dq8.compute_tables(qs.astype(np.float32))
    np.testing.assert_array_equal(t32[0], O.compute_tables(books8, qs[0].astype(np.float32)))


# ---------------------------------------------------------------- graph replay
def test_graph_never_replays_on_a_new_list():
    """Search a list twice (the device phase is captured as a CUDA graph),
    free it, create another list of the same size with other codes and an
    id offset, search it 4 times: every result is the new list's."""
    rng = np.random.default_rng(43)
    x = mixture(rng, 300_000, 64, comps=64)
    books = kmeans_books(x[:8000], 16, 16, iters=3)
    dq = P.DeviceQuantizer(P.ProductQuantizer(16, 4, 64, books))
    qs = x[:32] + 1.0
    n = 150_000
    a_codes, b_codes = encode(books, x[:n]), encode(books, x[n:2 * n])
    db = P.DeviceCodes(a_codes, 4)
    for _ in range(3):
        db.qadc_search(dq, qs, 200, 40)
    del db
    gc.collect()
    db2 = P.DeviceCodes(b_codes, 4, id_base=7_000_000)
    want = [O.qadc_scan(b_codes, np.arange(n) + 7_000_000, O.compute_tables(books, q), 200, 40)[:2] for q in qs]
    for _ in range(4):
        b, i, c, _, _ = db2.qadc_search(dq, qs, 200, 40)
        for qi in range(len(qs)):
            np.testing.assert_array_equal(b[qi], want[qi][0])
            np.testing.assert_array_equal(i[qi], want[qi][1])


def test_graph_sees_a_new_prefix():
    """pqs_db_set_prefix changes qmax: a captured graph must not replay."""
    rng = np.random.default_rng(44)
    x = mixture(rng, 200_000, 64, comps=64)
    books = kmeans_books(x[:8000], 16, 16, iters=3)
    dq = P.DeviceQuantizer(P.ProductQuantizer(16, 4, 64, books))
    codes = encode(books, x)
    qs = x[:16] + 1.0
    db = P.DeviceCodes(codes[100_000:], 4, id_base=100_000)
    for pre in (codes[:1000], codes[50_000:51_000]):
        db.set_prefix(pre)
        for _ in range(3):
            b, i, c, _, _ = db.qadc_search(dq, qs, 1000, 30)
        for qi, q in enumerate(qs):
            t = O.compute_tables(books, q)
            qmin, qmax = O.qadc_params(t, pre, 1000, 30)   # the global prefix (quickadc.py:129-137)
            dist = O.quantized_distances(codes[100_000:], O.quantize(qmin, qmax, t))
            ob, oi = O.select_best(dist.astype(np.float64), np.arange(100_000, 200_000), 30)
            np.testing.assert_array_equal(b[qi], ob.astype(np.uint8))
            np.testing.assert_array_equal(i[qi], oi)


# ---------------------------------------------------------------- cache coherence
def test_inplace_edit_refused_and_rebinding_reuploads():
    rng = np.random.default_rng(45)
    x = mixture(rng, 20_000, 32, comps=32)
    books = kmeans_books(x[:4000], 4, 256, iters=2)
    pq = P.ProductQuantizer(4, 8, 32, books)
    codes = encode(books, x)
    cl = P.CodeList(codes.copy())
    t = P.compute_tables(pq, x[0] + 1.0)
    first = P.scan(cl, t, 10).items()
    with pytest.raises(ValueError):
        cl.codes[0, 0] = 3          # the uploaded array is read-only now
    other = np.ascontiguousarray(codes[::-1])
    cl.codes = other               # rebinding: the next search re-uploads
    got = P.scan(cl, t, 10).items()
    od, oi = O.scan(other, np.arange(len(other)), t.tables, 10)
    assert got == list(zip(od.tolist(), oi.tolist()))
    assert got != first
    cl.ids = np.arange(len(other)) + 5   # new ids are honoured too
    got = P.scan(cl, t, 10).items()
    assert [i for _, i in got] == (oi + 5).tolist()


def test_ivf_list_replacement_reuploads():
    rng = np.random.default_rng(46)
    x = mixture(rng, 6000, 32, comps=16)
    books = kmeans_books(x[:3000], 4, 256, iters=2)
    pq = P.ProductQuantizer(4, 8, 32, books)
    coarse = x[:8].copy()
    assign = ((x[:, None, :] - coarse[None]) ** 2).sum(-1).argmin(1)
    codes = encode(books, x)
    lists_codes = [codes[assign == c] for c in range(8)]
    lists_ids = [np.flatnonzero(assign == c).astype(np.int64) for c in range(8)]
    idx = P.IvfIndex(coarse, pq, [P.CodeList(c, i) for c, i in zip(lists_codes, lists_ids)])
    q = x[5] + 0.5
    P.query_ivf(idx, q, ma=8, r=10)
    lists_codes[3] = lists_codes[3][::-1].copy()
    lists_ids[3] = lists_ids[3][::-1] + 100_000
    idx.lists[3] = P.CodeList(lists_codes[3], lists_ids[3])
    got = P.query_ivf(idx, q, ma=8, r=10).items()
    od, oi = O.query_ivf(coarse, books, lists_codes, lists_ids, q, 8, 10)
    assert got == list(zip(od.tolist(), oi.tolist()))
