"""Generate golden fixtures by running the REAL reference package.

Run in the build container (the reference is mounted read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `pqscan` from /root/reference, runs the hot-path functions on small
seeded inputs and stores inputs + outputs as .npz files next to this script.
The fixtures are committed; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import pqscan  # noqa: E402
from pqscan import (  # noqa: E402
    CodeList,
    LookupTables,
    QuantParams,
    QuantizedTables4,
    TrainConfig,
    build_ivf,
    compute_tables,
    encode,
    generate_synthetic,
    qadc_block,
    qadc_scan,
    quantize,
    quantized_distances,
    query_ivf,
    scan,
    scan_distances,
    train_pq,
    transpose_blocks,
)
from pqscan._dist import nearest_k  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, {k: v.shape for k, v in arrays.items()})


def items_arrays(nset, r):
    items = nset.items()
    d = np.full(r, np.nan)
    i = np.full(r, -1, dtype=np.int64)
    for p, (dist, ident) in enumerate(items):
        d[p] = dist
        i[p] = ident
    return d, i, len(items)


def mixture(rng, n, d, comps, hi, sigma, clip_lo=None, clip_hi=None):
    centers = rng.uniform(0.0, hi, size=(comps, d))
    lab = rng.integers(0, comps, size=n)
    x = centers[lab] + rng.normal(0.0, sigma, size=(n, d))
    if clip_lo is not None or clip_hi is not None:
        x = np.clip(x, clip_lo, clip_hi)
    return x.astype(np.float32)


def g_tables():
    """compute_tables bitwise, for three table shapes (cfg0/1/2-like)."""
    rng = np.random.default_rng(101)
    out = {}
    for tag, (d, m, b, hi, sigma) in {
        "c0": (128, 8, 8, 128.0, 16.0),
        "c1": (128, 16, 4, 128.0, 16.0),
        "c2": (960, 64, 8, 1.0, 0.05),
    }.items():
        x = mixture(rng, 3000, d, 16, hi, sigma, 0.0, 255.0)
        pq = train_pq(x[:2000], m, b, TrainConfig(kmeans_iters=4, seed=7))
        qs = x[2000:2006] + rng.normal(0, sigma / 2, (6, d)).astype(np.float32)
        tabs = np.stack([compute_tables(pq, q).tables for q in qs])
        out[f"{tag}_codebooks"] = pq.codebooks
        out[f"{tag}_queries"] = qs
        out[f"{tag}_tables"] = tabs
        codes = encode(pq, x[:500])
        out[f"{tag}_codes"] = codes
        out[f"{tag}_dist"] = np.stack([scan_distances(compute_tables(pq, q), codes) for q in qs])
    save("tables.npz", **out)


def g_scan():
    """scan() on random instances (criterion-9 style) incl. ties and r > n."""
    rng = np.random.default_rng(202)
    cases = []
    for trial in range(40):
        n = int(rng.integers(1, 600))
        m = int(rng.integers(1, 9))
        k = int(rng.integers(2, 257))
        r = int(rng.integers(1, n + 5))
        if trial % 5 == 0:
            # coarse tables -> many exact distance ties
            tables = rng.integers(0, 4, (m, k)).astype(np.float32)
        else:
            tables = (rng.random((m, k)) * 100).astype(np.float32)
        codes = rng.integers(0, k, (n, m)).astype(np.uint8)
        ids = rng.permutation(n * 3)[:n].astype(np.int64)
        nset = scan(CodeList(codes, ids), LookupTables(tables), r)
        d, i, cnt = items_arrays(nset, r)
        cases.append(dict(tables=tables, codes=codes, ids=ids, r=np.int64(r),
                          dist=d, out_ids=i, count=np.int64(cnt)))
    flat = {}
    for c, case in enumerate(cases):
        for key, val in case.items():
            flat[f"{c}_{key}"] = np.asarray(val)
    flat["ncases"] = np.int64(len(cases))
    save("scan.npz", **flat)


def g_quick_adc():
    """qadc_scan on trained 4-bit PQ data, several init_count / r."""
    rng = np.random.default_rng(303)
    x = mixture(rng, 6000, 64, 32, 128.0, 16.0, 0.0, 255.0)
    pq = train_pq(x[:3000], 16, 4, TrainConfig(kmeans_iters=6, seed=1))
    codes = encode(pq, x[:5000])
    ids = np.arange(5000, dtype=np.int64)
    tlist = transpose_blocks(CodeList(codes, ids), 4)
    qs = x[5000:5012] + rng.normal(0, 8, (12, 64)).astype(np.float32)
    out = dict(codebooks=pq.codebooks, codes=codes, queries=qs, blocks=tlist.blocks)
    settings = [(200, 100), (200, 10), (50, 100), (5000, 20), (1, 1), (7, 300)]
    for s, (init, r) in enumerate(settings):
        bins = np.full((len(qs), r), np.nan)
        oids = np.full((len(qs), r), -1, dtype=np.int64)
        qts = np.zeros((len(qs), 16, 16), dtype=np.uint8)
        qmm = np.zeros((len(qs), 2))
        for qi, q in enumerate(qs):
            tables = compute_tables(pq, q)
            nset, qt = qadc_scan(tlist, tables, init, r)
            d, i, _ = items_arrays(nset, r)
            bins[qi], oids[qi] = d, i
            qts[qi] = qt.tables
            qmm[qi] = (qt.params.qmin, qt.params.qmax)
        out[f"s{s}_init"] = np.int64(init)
        out[f"s{s}_r"] = np.int64(r)
        out[f"s{s}_bins"] = bins
        out[f"s{s}_ids"] = oids
        out[f"s{s}_qtables"] = qts
        out[f"s{s}_qminmax"] = qmm
    # permuted ids + tail padding (n not a multiple of 16)
    n2 = 1237
    ids2 = rng.permutation(10 * n2)[:n2].astype(np.int64)
    tl2 = transpose_blocks(CodeList(codes[:n2], ids2), 4)
    q = qs[0]
    nset, qt = qadc_scan(tl2, compute_tables(pq, q), 200, 64)
    d, i, _ = items_arrays(nset, 64)
    out.update(p_ids=ids2, p_bins=d, p_out_ids=i, p_qtables=qt.tables,
               p_qminmax=np.array([qt.params.qmin, qt.params.qmax]))
    save("quick_adc.npz", **out)


def g_quantize():
    """quantize boundaries + quantized_distances + qadc_block known answers."""
    rng = np.random.default_rng(404)
    vals = np.concatenate([
        np.array([0.0, 2.0, 7.9999, 8.0, 100.0, 1e-9, 3.99999]),
        rng.random(200) * 10,
    ])
    params = [(0.0, 8.0), (2.0, 10.0), (1.0, 1.0), (0.5, 9.75)]
    q = np.stack([quantize(QuantParams(a, b), vals) for a, b in params])
    qt = rng.integers(0, 128, (8, 16)).astype(np.uint8)
    codes = rng.integers(0, 16, (333, 8)).astype(np.uint8)
    qd = quantized_distances(codes, QuantizedTables4(qt, QuantParams(0.0, 127.0)))
    blocks = rng.integers(0, 256, (200, 4, 16)).astype(np.uint8)
    qb = np.stack([qadc_block(b, QuantizedTables4(qt, QuantParams(0.0, 127.0))) for b in blocks])
    save("quantize.npz", values=vals, params=np.array(params), bins=q,
         qtables=qt, codes=codes, qdist=qd, blocks=blocks, qblock=qb)


def g_ivf():
    """query_ivf (kernel='adc') on a small built index, ma in {1,4,16}."""
    rng = np.random.default_rng(505)
    base = mixture(rng, 4000, 32, 24, 128.0, 16.0, 0.0, 255.0)
    idx = build_ivf(base, K=32, m=4, b=8, cfg=TrainConfig(kmeans_iters=6, seed=2))
    qs = base[rng.choice(4000, 8, replace=False)] + rng.normal(0, 6, (8, 32)).astype(np.float32)
    out = dict(coarse=idx.coarse, codebooks=idx.pq.codebooks, queries=qs)
    sizes = np.array([lst.n for lst in idx.lists], dtype=np.int64)
    out["list_sizes"] = sizes
    out["list_codes"] = np.concatenate([lst.codes for lst in idx.lists])
    out["list_ids"] = np.concatenate([lst.ids for lst in idx.lists])
    for ma, r in [(1, 20), (4, 50), (16, 100), (32, 10)]:
        d = np.full((len(qs), r), np.nan)
        i = np.full((len(qs), r), -1, dtype=np.int64)
        for qi, q in enumerate(qs):
            dd, ii, _ = items_arrays(query_ivf(idx, q, ma=ma, r=r), r)
            d[qi], i[qi] = dd, ii
        out[f"ma{ma}_r{r}_dist"] = d
        out[f"ma{ma}_r{r}_ids"] = i
    cells, cd = nearest_k(qs.astype(np.float64), idx.coarse.astype(np.float64), 8)
    out["probe_cells"] = cells
    out["probe_dist"] = cd
    save("ivf.npz", **out)


def g_ivf_qadc():
    """query_ivf kernel='quick-adc' (ivf.py:185-190): a built 8x4 index (ids
    ascending per list) and a hand-made one with permuted ids, a small code
    alphabet (heavy bin ties), empty and tiny lists; init_count below r,
    between r and the list sizes, and above every list size."""
    from pqscan import IvfIndex, ProductQuantizer

    rng = np.random.default_rng(808)
    base = mixture(rng, 3000, 32, 16, 128.0, 16.0, 0.0, 255.0)
    idx = build_ivf(base, K=24, m=8, b=4, cfg=TrainConfig(kmeans_iters=5, seed=7))
    qs = base[rng.choice(3000, 6, replace=False)] + rng.normal(0, 6, (6, 32)).astype(np.float32)
    out = {}

    def dump(tag, index, settings):
        out[f"{tag}_coarse"] = index.coarse
        out[f"{tag}_codebooks"] = index.pq.codebooks
        out[f"{tag}_list_sizes"] = np.array([lst.n for lst in index.lists], dtype=np.int64)
        out[f"{tag}_list_codes"] = np.concatenate([lst.codes for lst in index.lists]).reshape(-1, index.pq.m)
        out[f"{tag}_list_ids"] = np.concatenate([lst.ids for lst in index.lists])
        for ma, r, ic in settings:
            d = np.full((len(qs), r), np.nan)
            i = np.full((len(qs), r), -1, dtype=np.int64)
            for qi, q in enumerate(qs):
                dd, ii, _ = items_arrays(query_ivf(index, q, ma=ma, r=r, kernel="quick-adc", init_count=ic), r)
                d[qi], i[qi] = dd, ii
            out[f"{tag}_ma{ma}_r{r}_i{ic}_dist"] = d
            out[f"{tag}_ma{ma}_r{r}_i{ic}_ids"] = i

    dump("built", idx, [(1, 20, 200), (4, 50, 30), (8, 100, 200), (24, 10, 5000)])
    # hand-made index: permuted ids, codes from a 3-symbol alphabet -> many equal bins
    K = 6
    coarse = base[rng.choice(3000, K, replace=False)]
    pq = ProductQuantizer(m=8, b=4, d=32, codebooks=idx.pq.codebooks)
    sizes = [700, 0, 3, 150, 1, 400]
    perm = rng.permutation(10_000)[: sum(sizes)].astype(np.int64)
    lists, o = [], 0
    for sz in sizes:
        codes = rng.integers(0, 3, (sz, 8)).astype(np.uint8)
        lists.append(CodeList(codes, perm[o:o + sz]))
        o += sz
    dump("ties", IvfIndex(coarse=coarse, pq=pq, lists=lists), [(6, 100, 200), (3, 40, 1), (2, 250, 64)])
    out["queries"] = qs
    save("ivf_qadc.npz", **out)


def g_fastscan():
    """fast_scan (fastscan.py:328-386) on a grouped 8x8 database: neighbour
    sets and ScanStats for several (init, r); a PQG1 file."""
    from pqscan import fast_scan, group_codes, save_grouped

    rng = np.random.default_rng(909)
    x = mixture(rng, 24000, 32, 24, 128.0, 16.0, 0.0, 255.0)
    pq = train_pq(x[:6000], 8, 8, TrainConfig(kmeans_iters=4, seed=8))
    codes = encode(pq, x[:20000])
    ids = rng.permutation(50_000)[:20000].astype(np.int64)
    grouped = group_codes(CodeList(codes, ids))
    qs = x[20000:20006] + rng.normal(0, 4, (6, 32)).astype(np.float32)
    out = dict(codebooks=pq.codebooks, codes=codes, ids=ids, queries=qs,
               g_keys=grouped.keys, g_offsets=grouped.offsets, g_counts=grouped.counts,
               g_packed=grouped.packed, g_ids=grouped.ids)
    for init, r in [(0.01, 100), (0.05, 10), (0.001, 1), (1.0, 50), (0.0002, 300)]:
        tag = f"i{init}_r{r}"
        d = np.full((len(qs), r), np.nan)
        i = np.full((len(qs), r), -1, dtype=np.int64)
        st = np.zeros((len(qs), 3), dtype=np.int64)
        for qi, q in enumerate(qs):
            nset, stats = fast_scan(grouped, compute_tables(pq, q), init, r)
            d[qi], i[qi], _ = items_arrays(nset, r)
            st[qi] = (stats.total, stats.checked, stats.pruned)
        out[f"{tag}_dist"], out[f"{tag}_ids"], out[f"{tag}_stats"] = d, i, st
    save_grouped(os.path.join(OUT, "fmt_grouped.pqg"), group_codes(CodeList(codes[:300], ids[:300])))
    save("fastscan.npz", **out)


def g_derived():
    """search_two_pass (derived.py:402-409) on a trained DerivedPQ, query_ivf
    kernel='derived' on a built index with a derived quantizer, and the
    PQZ1+derived / IVF1+derived files."""
    from pqscan import build_ivf, save_derived, save_ivf, search_two_pass, train_derived

    rng = np.random.default_rng(1010)
    x = mixture(rng, 9000, 32, 16, 128.0, 16.0, 0.0, 255.0)
    dpq = train_derived(x[:4000], 8, 8, 4, TrainConfig(kmeans_iters=3, seed=11))
    codes = encode(dpq.pq, x[:6000])
    ids = rng.permutation(20_000)[:6000].astype(np.int64)
    qs = x[6000:6005] + rng.normal(0, 4, (5, 32)).astype(np.float32)
    out = dict(books=dpq.pq.codebooks, derived=dpq.derived, codes=codes, ids=ids, queries=qs)
    for r, r2 in [(10, 50), (100, 9000), (5, 1), (20, 300), (50, 6000)]:
        d = np.full((len(qs), r), np.nan)
        i = np.full((len(qs), r), -1, dtype=np.int64)
        for qi, q in enumerate(qs):
            d[qi], i[qi], _ = items_arrays(search_two_pass(dpq, CodeList(codes, ids), q, r, r2), r)
        out[f"r{r}_r2{r2}_dist"], out[f"r{r}_r2{r2}_ids"] = d, i
    save_derived(os.path.join(OUT, "fmt_derived.pqz"), dpq)
    idx = build_ivf(x[:5000], K=12, m=8, b=8, cfg=TrainConfig(kmeans_iters=3, seed=12), bderived=3)
    out["ivf_coarse"], out["ivf_books"], out["ivf_derived"] = idx.coarse, idx.pq.codebooks, idx.dpq.derived
    out["ivf_sizes"] = np.array([l.n for l in idx.lists], np.int64)
    out["ivf_codes"] = np.concatenate([l.codes for l in idx.lists])
    out["ivf_ids"] = np.concatenate([l.ids for l in idx.lists])
    for ma, r, r2 in [(3, 20, 100), (12, 50, None), (2, 10, 1)]:
        d = np.full((len(qs), r), np.nan)
        i = np.full((len(qs), r), -1, dtype=np.int64)
        for qi, q in enumerate(qs):
            d[qi], i[qi], _ = items_arrays(query_ivf(idx, q, ma=ma, r=r, kernel="derived", r2=r2), r)
        out[f"ivf_ma{ma}_r{r}_r2{r2}_dist"], out[f"ivf_ma{ma}_r{r}_r2{r2}_ids"] = d, i
    save_ivf(os.path.join(OUT, "fmt_index_derived.ivf"), build_ivf(x[:1500], K=4, m=4, b=6,
             cfg=TrainConfig(kmeans_iters=2, seed=13), bderived=2))
    save("derived.npz", **out)


def g_encode():
    """encode (plain and IVF-residual) incl. exact centroid ties."""
    rng = np.random.default_rng(606)
    out = {}
    for tag, (d, m, b, hi, sigma, nx) in {
        "c1": (96, 16, 4, 1.0, 0.3, 600),
        "c3": (128, 8, 8, 128.0, 16.0, 600),
        "c2": (960, 64, 8, 1.0, 0.05, 150),
    }.items():
        x = mixture(rng, 1500 + nx, d, 12, hi, sigma, 0.0, 255.0)
        pq = train_pq(x[:1500], m, b, TrainConfig(kmeans_iters=3, seed=3))
        books = pq.codebooks.copy()
        books[:, -1] = books[:, 0]           # duplicate centroid -> exact ties
        pq = type(pq)(m=m, b=b, d=d, codebooks=books)
        xs = x[1500:].copy()
        xs[:50] = books[:, 0].reshape(-1)    # rows exactly on the tied centroid
        out[f"{tag}_codebooks"] = books
        out[f"{tag}_x"] = xs
        out[f"{tag}_codes"] = encode(pq, xs)
        coarse = x[rng.choice(1500, 40, replace=False)].astype(np.float32)
        cells = rng.integers(0, 40, xs.shape[0]).astype(np.int64)
        res = xs.astype(np.float64) - coarse[cells].astype(np.float64)
        out[f"{tag}_coarse"] = coarse
        out[f"{tag}_cells"] = cells
        out[f"{tag}_rescodes"] = encode(pq, res)
    save("encode.npz", **out)


def g_fp64():
    """float64 queries / vectors that float32 cannot represent (the reference
    computes from float64(query): quantizer.py:85-89, ivf.py:170, encode
    quantizer.py:319-323): tables, scan, qadc_scan, query_ivf ('adc' and
    'quick-adc'), the probes and encode."""
    rng = np.random.default_rng(707)
    base = mixture(rng, 5000, 32, 24, 128.0, 16.0, 0.0, 255.0)
    qs = (base[rng.choice(5000, 6, replace=False)].astype(np.float64)
          + rng.normal(0.0, 6.0, (6, 32)))          # fp64, not fp32-representable
    assert not np.array_equal(qs.astype(np.float32).astype(np.float64), qs)
    out = dict(queries=qs)
    pq8 = train_pq(base[:3000], 4, 8, TrainConfig(kmeans_iters=4, seed=4))
    codes8 = encode(pq8, base)
    out.update(pq8_books=pq8.codebooks, codes8=codes8)
    pq4 = train_pq(base[:3000], 8, 4, TrainConfig(kmeans_iters=4, seed=5))
    codes4 = encode(pq4, base)
    out.update(pq4_books=pq4.codebooks, codes4=codes4)
    tl = transpose_blocks(CodeList(codes4), 4)
    t8, s_d, s_i, q_b, q_i = [], [], [], [], []
    for q in qs:
        t = compute_tables(pq8, q)
        t8.append(t.tables)
        d, i, _ = items_arrays(scan(CodeList(codes8), t, 20), 20)
        s_d.append(d)
        s_i.append(i)
        nset, _ = qadc_scan(tl, compute_tables(pq4, q), 200, 30)
        d, i, _ = items_arrays(nset, 30)
        q_b.append(d)
        q_i.append(i)
    out.update(tables8=np.stack(t8), scan_dist=np.stack(s_d), scan_ids=np.stack(s_i), qadc_bins=np.stack(q_b),
               qadc_ids=np.stack(q_i))
    idx = build_ivf(base, K=32, m=4, b=8, cfg=TrainConfig(kmeans_iters=6, seed=2))
    out.update(coarse=idx.coarse, ivf_books=idx.pq.codebooks,
               list_sizes=np.array([lst.n for lst in idx.lists], dtype=np.int64),
               list_codes=np.concatenate([lst.codes for lst in idx.lists]),
               list_ids=np.concatenate([lst.ids for lst in idx.lists]))
    d, i = zip(*[items_arrays(query_ivf(idx, q, ma=5, r=25), 25)[:2] for q in qs])
    out.update(ivf_dist=np.stack(d), ivf_ids=np.stack(i))
    cells, cd = nearest_k(qs, idx.coarse.astype(np.float64), 7)
    out.update(probe_cells=cells, probe_dist=cd)
    idx4 = build_ivf(base, K=16, m=8, b=4, cfg=TrainConfig(kmeans_iters=4, seed=3))
    out.update(coarse4=idx4.coarse, ivf4_books=idx4.pq.codebooks,
               list4_sizes=np.array([lst.n for lst in idx4.lists], dtype=np.int64),
               list4_codes=np.concatenate([lst.codes for lst in idx4.lists]),
               list4_ids=np.concatenate([lst.ids for lst in idx4.lists]))
    d, i = zip(*[items_arrays(query_ivf(idx4, q, ma=3, r=15, kernel="quick-adc", init_count=50), 15)[:2] for q in qs])
    out.update(ivfq_dist=np.stack(d), ivfq_ids=np.stack(i))
    xs = base[:200].astype(np.float64) + rng.normal(0.0, 1e-3, (200, 32))
    out.update(enc_x=xs, enc_codes=encode(pq8, xs))
    save("fp64.npz", **out)


def g_formats():
    """PQZ1 / PQL1 (b = 4 packed nibbles, b = 8) / IVF1 files written by the reference."""
    from pqscan import save_codes, save_ivf, save_quantizer

    rng = np.random.default_rng(707)
    x = mixture(rng, 3000, 32, 8, 128.0, 16.0, 0.0, 255.0)
    pq8 = train_pq(x[:2000], 4, 8, TrainConfig(kmeans_iters=2, seed=4))
    pq4 = train_pq(x[:2000], 8, 4, TrainConfig(kmeans_iters=2, seed=5))
    save_quantizer(os.path.join(OUT, "fmt_pq8.pqz"), pq8)
    save_quantizer(os.path.join(OUT, "fmt_pq4.pqz"), pq4)
    c8 = encode(pq8, x[:777])
    c4 = encode(pq4, x[:555])
    ids = rng.permutation(5000)[:777].astype(np.int64)
    save_codes(os.path.join(OUT, "fmt_codes8.pql"), CodeList(c8, ids), 8)
    save_codes(os.path.join(OUT, "fmt_codes4.pql"), CodeList(c4), 4)
    c3 = rng.integers(0, 8, (101, 5)).astype(np.uint8)             # odd m, b = 3 (nibble packed)
    save_codes(os.path.join(OUT, "fmt_codes3.pql"), CodeList(c3), 3)
    idx = build_ivf(x[:2500], K=16, m=4, b=8, cfg=TrainConfig(kmeans_iters=2, seed=6))
    save_ivf(os.path.join(OUT, "fmt_index.ivf"), idx)
    save("formats.npz", pq8_books=pq8.codebooks, pq4_books=pq4.codebooks, codes8=c8, ids8=ids, codes4=c4, codes3=c3,
         ivf_coarse=idx.coarse, ivf_books=idx.pq.codebooks,
         ivf_sizes=np.array([l.n for l in idx.lists], np.int64),
         ivf_codes=np.concatenate([l.codes for l in idx.lists]),
         ivf_ids=np.concatenate([l.ids for l in idx.lists]))


if __name__ == "__main__":
    print("pqscan from", pqscan.__file__)
    if len(sys.argv) > 1:            # regenerate selected fixtures only
        for name in sys.argv[1:]:
            globals()[f"g_{name}"]()
        sys.exit(0)
    g_tables()
    g_scan()
    g_quick_adc()
    g_quantize()
    g_ivf()
    g_ivf_qadc()
    g_fastscan()
    g_derived()
    g_encode()
    g_fp64()
    g_formats()
