"""GPU parity: libpqs.so vs the golden fixtures (real reference outputs) and
the CPU oracle on seeded inputs.  Bar: bit-exact (tables, fp64 distances,
bins, ids); the float path's fp64 distances are bit-identical to the
reference because candidates are re-scored in its summation order."""

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


# ---------------------------------------------------------------- golden
@pytest.mark.parametrize("tag", ["c0", "c1", "c2"])
def test_tables_bitwise(golden, tag):
    g = golden("tables.npz")
    books, qs = g[f"{tag}_codebooks"], g[f"{tag}_queries"]
    m, k, dsub = books.shape
    pq = P.ProductQuantizer(m, int(np.log2(k)), m * dsub, books)
    got = P.compute_tables_batch(pq, qs)
    np.testing.assert_array_equal(got.view(np.uint32), g[f"{tag}_tables"].view(np.uint32))
    one = P.compute_tables(pq, qs[0]).tables
    np.testing.assert_array_equal(one.view(np.uint32), g[f"{tag}_tables"][0].view(np.uint32))


@pytest.mark.parametrize("tag", ["c0", "c1", "c2"])
def test_scan_distances_bitwise(golden, tag):
    g = golden("tables.npz")
    for qi in range(g[f"{tag}_tables"].shape[0]):
        got = P.scan_distances(P.LookupTables(g[f"{tag}_tables"][qi]), g[f"{tag}_codes"])
        np.testing.assert_array_equal(got, g[f"{tag}_dist"][qi])


def test_scan_golden_cases(golden):
    g = golden("scan.npz")
    for c in range(int(g["ncases"])):
        r = int(g[f"{c}_r"])
        cl = P.CodeList(g[f"{c}_codes"], g[f"{c}_ids"])
        got = P.scan(cl, P.LookupTables(g[f"{c}_tables"]), r).items()
        cnt = int(g[f"{c}_count"])
        want = list(zip(g[f"{c}_dist"][:cnt].tolist(), g[f"{c}_out_ids"][:cnt].tolist()))
        assert got == want, f"case {c}"


def test_quick_adc_golden(golden):
    g = golden("quick_adc.npz")
    books = g["codebooks"]
    pq = P.ProductQuantizer(16, 4, 64, books)
    tl = P.transpose_blocks(P.CodeList(g["codes"]), 4)
    for s in range(6):
        init, r = int(g[f"s{s}_init"]), int(g[f"s{s}_r"])
        for qi, q in enumerate(g["queries"]):
            nset, qt = P.qadc_scan(tl, P.compute_tables(pq, q), init, r)
            items = nset.items()
            n = len(items)
            assert [d for d, _ in items] == g[f"s{s}_bins"][qi][:n].tolist()
            assert [i for _, i in items] == g[f"s{s}_ids"][qi][:n].tolist()
            np.testing.assert_array_equal(qt.tables, g[f"s{s}_qtables"][qi])
            assert (qt.params.qmin, qt.params.qmax) == tuple(g[f"s{s}_qminmax"][qi])


def test_quick_adc_permuted_ids_padding(golden):
    g = golden("quick_adc.npz")
    pq = P.ProductQuantizer(16, 4, 64, g["codebooks"])
    n2 = g["p_ids"].shape[0]
    tl = P.transpose_blocks(P.CodeList(g["codes"][:n2], g["p_ids"]), 4)
    nset, qt = P.qadc_scan(tl, P.compute_tables(pq, g["queries"][0]), 200, 64)
    assert [d for d, _ in nset.items()] == g["p_bins"].tolist()
    assert [i for _, i in nset.items()] == g["p_out_ids"].tolist()
    np.testing.assert_array_equal(qt.tables, g["p_qtables"])


def test_quantize_golden(golden):
    g = golden("quantize.npz")
    for p, (a, b) in enumerate(g["params"]):
        np.testing.assert_array_equal(P.quantize(P.QuantParams(a, b), g["values"]), g["bins"][p])
    qt = P.QuantizedTables4(g["qtables"], P.QuantParams(0.0, 127.0))
    np.testing.assert_array_equal(P.quantized_distances(g["codes"], qt), g["qdist"])
    for bi in range(0, g["blocks"].shape[0], 7):
        np.testing.assert_array_equal(P.qadc_block(g["blocks"][bi], qt), g["qblock"][bi])
    assert P.quantize(P.QuantParams(0.0, 8.0), 7.9999) == 126
    assert P.quantize(P.QuantParams(0.0, 8.0), 8.0) == 127


def _golden_ivf(g):
    pq = P.ProductQuantizer(4, 8, 32, g["codebooks"])
    sizes = g["list_sizes"]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    lists = [P.CodeList(g["list_codes"][offs[c]:offs[c + 1]], g["list_ids"][offs[c]:offs[c + 1]])
             for c in range(len(sizes))]
    return P.IvfIndex(g["coarse"], pq, lists)


def test_ivf_probes_golden(golden):
    g = golden("ivf.npz")
    idx = _golden_ivf(g)
    dev = P.ivf.device_index(idx)
    cells, dist = dev.probe(g["queries"], 8)
    np.testing.assert_array_equal(cells, g["probe_cells"])
    np.testing.assert_array_equal(dist, g["probe_dist"])


@pytest.mark.parametrize("ma,r", [(1, 20), (4, 50), (16, 100), (32, 10)])
def test_ivf_golden(golden, ma, r):
    g = golden("ivf.npz")
    idx = _golden_ivf(g)
    for qi, q in enumerate(g["queries"]):
        items = P.query_ivf(idx, q, ma=ma, r=r).items()
        n = len(items)
        assert [d for d, _ in items] == g[f"ma{ma}_r{r}_dist"][qi][:n].tolist()
        assert [i for _, i in items] == g[f"ma{ma}_r{r}_ids"][qi][:n].tolist()


# ------------------------------------------------------ larger vs oracle
@pytest.fixture(scope="module")
def data4():
    rng = np.random.default_rng(7)
    x = mixture(rng, 150_000, 64, comps=64)
    books = kmeans_books(x[:20000], 16, 16, iters=5)
    codes = encode(books, x)
    qs = mixture(np.random.default_rng(8), 24, 64, comps=64)
    return books, codes, qs


def _qadc_oracle(books, codes, ids, q, init, r):
    t = O.compute_tables(books, q)
    return O.qadc_scan(codes, ids, t, init, r)


@pytest.mark.parametrize("init,r", [(200, 100), (1000, 10), (50, 7)])
def test_qadc_batched_vs_oracle(data4, init, r):
    """150k codes > candidate cap: exercises the sampled threshold path."""
    books, codes, qs = data4
    pq = P.ProductQuantizer(16, 4, 64, books)
    dq = P.DeviceQuantizer(pq)
    db = P.DeviceCodes(codes, 4)
    bins, ids, cnt, qt, qmm = db.qadc_search(dq, qs, init, r, want_tables=True)
    ctx = P.default_context()
    assert ctx.stat(3) == 0  # no fallback needed
    all_ids = np.arange(codes.shape[0], dtype=np.int64)
    for qi in range(0, len(qs), 4):
        ob, oi, oqt, qmin, qmax = _qadc_oracle(books, codes, all_ids, qs[qi], init, r)
        assert cnt[qi] == len(ob)
        np.testing.assert_array_equal(bins[qi, :cnt[qi]], ob.astype(np.uint8))
        np.testing.assert_array_equal(ids[qi, :cnt[qi]], oi)
        np.testing.assert_array_equal(qt[qi], oqt)
        assert (qmm[qi, 0], qmm[qi, 1]) == (qmin, qmax)


@pytest.mark.parametrize("mode", ["fallback", "tiny_cap"])
def test_qadc_fallback_paths(data4, mode):
    books, codes, qs = data4
    pq = P.ProductQuantizer(16, 4, 64, books)
    ctx = P.Context(0)
    dq = P.DeviceQuantizer(pq, ctx)
    db = P.DeviceCodes(codes[:60000], 4, ctx=ctx)
    if mode == "fallback":
        ctx.set_option(3, 1)
    else:
        ctx.set_option(1, 300)  # candidate cap below the tie counts -> overflow
    bins, ids, cnt, _, _ = db.qadc_search(dq, qs[:6], 200, 100)
    assert ctx.stat(3) > 0
    all_ids = np.arange(60000, dtype=np.int64)
    for qi in range(6):
        ob, oi, _, _, _ = _qadc_oracle(books, codes[:60000], all_ids, qs[qi], 200, 100)
        np.testing.assert_array_equal(bins[qi, :cnt[qi]], ob.astype(np.uint8))
        np.testing.assert_array_equal(ids[qi, :cnt[qi]], oi)


@pytest.fixture(scope="module")
def data8():
    rng = np.random.default_rng(17)
    x = mixture(rng, 120_000, 128)
    books = kmeans_books(x[:30000], 8, 256, iters=3)
    codes = encode(books, x)
    qs = mixture(np.random.default_rng(18), 16, 128)
    return books, codes, qs


@pytest.mark.parametrize("r", [100, 1, 777])
def test_adc_batched_vs_oracle(data8, r):
    books, codes, qs = data8
    pq = P.ProductQuantizer(8, 8, 128, books)
    dq = P.DeviceQuantizer(pq)
    db = P.DeviceCodes(codes, 8)
    d, i, c = db.adc_search(dq, qs, r)
    ids = np.arange(codes.shape[0], dtype=np.int64)
    for qi in range(0, len(qs), 3):
        od, oi = O.scan(codes, ids, O.compute_tables(books, qs[qi]), r)
        assert c[qi] == len(od)
        np.testing.assert_array_equal(d[qi, :c[qi]], od)
        np.testing.assert_array_equal(i[qi, :c[qi]], oi)


def test_adc_fallback_and_explicit_ids(data8):
    books, codes, qs = data8
    rng = np.random.default_rng(3)
    n = 50000
    ids = rng.permutation(10 * n)[:n].astype(np.int64)
    ctx = P.Context(0)
    ctx.set_option(3, 1)
    pq = P.ProductQuantizer(8, 8, 128, books)
    dq = P.DeviceQuantizer(pq, ctx)
    db = P.DeviceCodes(codes[:n], 8, ids=ids, ctx=ctx)
    d, i, c = db.adc_search(dq, qs[:4], 50)
    for qi in range(4):
        od, oi = O.scan(codes[:n], ids, O.compute_tables(books, qs[qi]), 50)
        np.testing.assert_array_equal(d[qi], od)
        np.testing.assert_array_equal(i[qi], oi)


def test_high_dim_m64(golden):
    """cfg2 shape family: m=64 sub-spaces, 15-dim sub-vectors."""
    g = golden("tables.npz")
    books = g["c2_codebooks"]
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 256, (40000, 64)).astype(np.uint8)
    qs = g["c2_queries"]
    pq = P.ProductQuantizer(64, 8, 960, books)
    db = P.DeviceCodes(codes, 8)
    d, i, c = db.adc_search(P.DeviceQuantizer(pq), qs, 100)
    ids = np.arange(40000, dtype=np.int64)
    for qi in range(len(qs)):
        od, oi = O.scan(codes, ids, O.compute_tables(books, qs[qi]), 100)
        np.testing.assert_array_equal(d[qi], od)
        np.testing.assert_array_equal(i[qi], oi)


def test_merge_equals_unsharded(data4):
    """Sharded Quick ADC with a global prefix == unsharded."""
    books, codes, qs = data4
    pq = P.ProductQuantizer(16, 4, 64, books)
    dq = P.DeviceQuantizer(pq)
    full = P.DeviceCodes(codes, 4)
    fb, fi, fc, _, _ = full.qadc_search(dq, qs, 200, 100)
    G = 3
    bounds = np.linspace(0, codes.shape[0], G + 1).astype(int)
    parts = []
    for g in range(G):
        sh = P.DeviceCodes(codes[bounds[g]:bounds[g + 1]], 4, id_base=int(bounds[g]))
        sh.set_prefix(codes[:200])
        parts.append(sh.qadc_search(dq, qs, 200, 100))
    dists = np.stack([p[0].astype(np.float64) for p in parts])
    dists[np.stack([p[1] for p in parts]) < 0] = np.inf
    ids = np.stack([p[1] for p in parts])
    cnts = np.stack([p[2] for p in parts])
    md, mi, mc = P.merge_topr(dists, ids, cnts, 100)
    np.testing.assert_array_equal(mc, fc)
    np.testing.assert_array_equal(mi, fi)
    np.testing.assert_array_equal(md.astype(np.uint8), fb)


def test_search_into_caller_buffers():
    """qadc_search / adc_search write into caller-owned (pinned) host buffers
    exactly what they return otherwise; bad buffers are refused."""
    import torch

    rng = np.random.default_rng(12)
    x = mixture(rng, 20000, 32, comps=16)
    books4 = kmeans_books(x[:4000], 8, 16, iters=3)
    books8 = kmeans_books(x[:4000], 4, 256, iters=2)
    qs = x[:9] + 1.0
    db4 = P.DeviceCodes(encode(books4, x), 4)
    dq4 = P.DeviceQuantizer(P.ProductQuantizer(8, 4, 32, books4))
    ref = db4.qadc_search(dq4, qs, 200, 50)
    out = (torch.empty((9, 50), dtype=torch.uint8).pin_memory().numpy(),
           torch.empty((9, 50), dtype=torch.int64).pin_memory().numpy(),
           torch.empty((9,), dtype=torch.int32).pin_memory().numpy())
    got = db4.qadc_search(dq4, qs, 200, 50, out=out)
    for a, b in zip(ref[:3], got[:3]):
        np.testing.assert_array_equal(a, b)
    assert got[0] is out[0]
    db8 = P.DeviceCodes(encode(books8, x), 8)
    dq8 = P.DeviceQuantizer(P.ProductQuantizer(4, 8, 32, books8))
    ref8 = db8.adc_search(dq8, qs, 20)
    out8 = (np.empty((9, 20)), np.empty((9, 20), np.int64), np.empty(9, np.int32))
    got8 = db8.adc_search(dq8, qs, 20, out=out8)
    for a, b in zip(ref8, got8):
        np.testing.assert_array_equal(a, b)
    with pytest.raises(ValueError):
        db8.adc_search(dq8, qs, 20, out=(np.empty((9, 20), np.float32), out8[1], out8[2]))
