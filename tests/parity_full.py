"""Full-size oracle parity over every query of the BASELINE configs.

    python tests/parity_full.py [cfg0 cfg1 cfg2 cfg3 cfg4] [--out profiles/parity_full_rNN.json]

For each config the device path runs the bench's own workload (same data,
same query batch) and is compared with the CPU oracle (oracle/; the numpy
restatement pinned to the real reference's outputs, and for the billion-code
config its C restatement oracle/qadc_oracle.c, pinned the same way) on:
  cfg0, cfg1, cfg2   all 1,000 queries (scan.py:197-203 / quickadc.py:104-141)
  cfg3               all 10,000 queries at the config's Q = 10,000 batch
                     (query_ivf kernel='adc', ivf.py:148-196)
  cfg4               1e9 codes as 8 shards of 125M (ids offset per shard, the
                     GLOBAL prefix of the first 1,000 codes): sharded + merged
                     == unsharded for all 10,000 queries, and a seeded sample
                     of queries against the oracle over all 1e9 codes
Bar: ids and fp64 distances / bins identical, every query.  The oracle runs
in a fork process pool over the host's cores.  Test infrastructure: lives in
tests/ (the only place besides smoke() and bench.py's CPU leg that may call
the oracle).
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

_W = {}


def _pool():
    return mp.get_context("fork").Pool(len(os.sched_getaffinity(0)))


def _scan_one(qi):
    from oracle import pqscan_oracle as O

    w = _W
    t = O.compute_tables(w["books"], w["queries"][qi])
    if w["b"] == 4:
        b, i, _, _, _ = O.qadc_scan(w["codes"], w["ids"], t, w["init"], w["r"])
        return b, i
    return O.scan(w["codes"], w["ids"], t, w["r"])


def _compare(got_d, got_i, got_c, want):
    bad = []
    for qi, (d, i) in enumerate(want):
        n = len(d)
        ok = int(got_c[qi]) == n and np.array_equal(np.asarray(got_d[qi][:n], np.float64), np.asarray(d, np.float64)) \
            and np.array_equal(got_i[qi][:n], i)
        if not ok:
            bad.append(qi)
    return bad


def exhaustive(name):
    import torch

    import paper_1712_02912_b200 as P
    from paper_1712_02912_b200 import datagen as G

    cfg = G.CONFIGS[name]
    t0 = time.time()
    books, codes, queries = G.make_exhaustive(name)
    pq = P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], books)
    dq = P.DeviceQuantizer(pq)
    db = P.DeviceCodes(codes, cfg["b"])
    if cfg["b"] == 4:
        d, i, c, _, _ = db.qadc_search(dq, queries, cfg["init_count"], cfg["r"])
    else:
        d, i, c = db.adc_search(dq, queries, cfg["r"])
    torch.cuda.synchronize()
    _W.clear()
    _W.update(books=books, codes=codes, queries=queries, ids=np.arange(codes.shape[0], dtype=np.int64), b=cfg["b"],
              init=cfg.get("init_count", 200), r=cfg["r"])
    with _pool() as pool:
        want = pool.map(_scan_one, range(queries.shape[0]), chunksize=4)
    bad = _compare(d, i, c, want)
    return {"config": name, "queries_checked": int(queries.shape[0]), "queries_in_batch": int(queries.shape[0]),
            "codes": int(codes.shape[0]), "mismatched_queries": bad, "mismatches": len(bad),
            "compared": "fp64 distances and ids" if cfg["b"] == 8 else "bins and ids",
            "oracle": "oracle/pqscan_oracle.py " + ("scan" if cfg["b"] == 8 else "qadc_scan"),
            "seconds": round(time.time() - t0, 1)}


def _ivf_one(qi):
    from oracle import pqscan_oracle as O

    w = _W
    return O.query_ivf(w["coarse"], w["books"], w["lists_codes"], w["lists_ids"], w["queries"][qi], w["ma"], w["r"])


def ivf():
    import torch

    import paper_1712_02912_b200 as P
    from paper_1712_02912_b200 import datagen as G

    cfg = G.CONFIGS["cfg3"]
    t0 = time.time()
    ctx = P.default_context()
    books, coarse, sizes, codes, ids, queries = G.make_ivf_device(
        "cfg3", lambda b: P.DeviceQuantizer(P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], b), ctx))
    pq = P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], books)
    ivf_ = P.DeviceIvf.from_arrays(pq, coarse, sizes, codes, ids, ctx=ctx)
    d, i, c = ivf_.search(queries, cfg["nprobe"], cfg["r"])     # the whole Q = 10,000 batch
    torch.cuda.synchronize()
    build_s = time.time() - t0
    codes_h, ids_h, coarse_h = codes.cpu().numpy(), ids.cpu().numpy(), coarse.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(sizes)])
    _W.clear()
    _W.update(books=books, coarse=coarse_h, queries=queries, ma=cfg["nprobe"], r=cfg["r"],
              lists_codes=[codes_h[offs[k]:offs[k + 1]] for k in range(len(sizes))],
              lists_ids=[ids_h[offs[k]:offs[k + 1]] for k in range(len(sizes))])
    with _pool() as pool:
        want = pool.map(_ivf_one, range(queries.shape[0]), chunksize=16)
    bad = _compare(d, i, c, want)
    return {"config": "cfg3", "queries_checked": int(queries.shape[0]), "queries_in_batch": int(queries.shape[0]),
            "codes": int(codes_h.shape[0]), "K": int(coarse_h.shape[0]), "nprobe": cfg["nprobe"],
            "mismatched_queries": bad, "mismatches": len(bad), "compared": "fp64 distances and ids",
            "oracle": "oracle/pqscan_oracle.py query_ivf", "index_build_s": round(build_s, 1),
            "seconds": round(time.time() - t0, 1)}


def _q4_one(qi):
    from oracle import c_oracle as C
    from oracle import pqscan_oracle as O

    w = _W
    t = O.compute_tables(w["books"], w["queries"][qi])
    qmin, qmax = O.qadc_params(t, w["prefix"], w["init"], w["r"])   # the global prefix (quickadc.py:129-137)
    qt = O.quantize(qmin, qmax, t)
    return C.qadc_topr(w["packed"], 16, qt, w["r"], id_base=0, scratch=True)


def billion(n_oracle_queries: int = 64, shards: int = 8, n_per: int | None = None):
    import torch

    import paper_1712_02912_b200 as P
    from paper_1712_02912_b200 import datagen as G

    cfg = G.CONFIGS["cfg4"]
    n_per = n_per or cfg["N"] // shards
    r, init = cfg["r"], cfg["init_count"]
    t0 = time.time()
    ctx = P.default_context()
    train = G.rows(cfg, 1712, 0, 100_000, stream=0)
    books = G.train_pq(train, cfg["m"], cfg["b"], iters=20, seed=1712)
    pq = P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], books)
    dq = P.DeviceQuantizer(pq, ctx)
    queries = G.rows(cfg, 1712, 0, cfg["Q"], stream=2)
    qd = torch.from_numpy(queries).cuda()
    prefix = G.device_encode_rows(dq, cfg, 1712, 0, init, stream=1)
    n_tot = n_per * shards
    packed = np.empty((n_tot, cfg["m"] // 2), np.uint8)
    parts = []
    all_codes = torch.empty((n_tot, cfg["m"]), dtype=torch.uint8, device="cuda")
    for s in range(shards):
        codes = G.device_encode_rows(dq, cfg, 1712, s * n_per, (s + 1) * n_per, stream=1)
        all_codes[s * n_per:(s + 1) * n_per] = codes
        packed[s * n_per:(s + 1) * n_per] = (codes[:, 0::2] | (codes[:, 1::2] << 4)).cpu().numpy()
        db = P.DeviceCodes(codes, 4, id_base=s * n_per, ctx=ctx)
        db.set_prefix(prefix)
        b, i, c, _, _ = db.qadc_search(dq, qd, init, r)
        parts.append((b.to(torch.float64), i, c))
        del db, codes
        torch.cuda.empty_cache()
    gd = torch.stack([p[0] for p in parts])
    gi = torch.stack([p[1] for p in parts])
    gc = torch.stack([p[2] for p in parts])
    md, mi, mc = P.merge_topr(gd, gi, gc, r, ctx=ctx)
    dball = P.DeviceCodes(all_codes, 4, ctx=ctx)   # the unsharded list (its own first codes are the prefix)
    del all_codes
    torch.cuda.empty_cache()
    ub, ui, uc, _, _ = dball.qadc_search(dq, qd, init, r)
    torch.cuda.synchronize()
    md, mi, mc = md.cpu().numpy(), mi.cpu().numpy(), mc.cpu().numpy()
    ub, ui, uc = ub.cpu().numpy(), ui.cpu().numpy(), uc.cpu().numpy()
    shard_bad = [q for q in range(queries.shape[0])
                 if not (mc[q] == uc[q] and np.array_equal(md[q].astype(np.uint8), ub[q])
                         and np.array_equal(mi[q], ui[q]))]
    gpu_s = time.time() - t0
    rng = np.random.default_rng(20261020)
    sample = np.sort(rng.choice(queries.shape[0], n_oracle_queries, replace=False))
    _W.clear()
    _W.update(books=books, queries=queries, prefix=prefix.cpu().numpy(), packed=packed, init=init, r=r)
    with _pool() as pool:
        want = pool.map(_q4_one, [int(q) for q in sample], chunksize=1)
    bad = [int(q) for q, (b, i) in zip(sample, want)
           if not (np.array_equal(ub[q][:len(b)], b) and np.array_equal(ui[q][:len(b)], i) and uc[q] == len(b))]
    ids_per_shard = {s: int(((ui[sample] >= s * n_per) & (ui[sample] < (s + 1) * n_per)).sum()) for s in range(shards)}
    return {"config": "cfg4", "codes": int(n_tot), "shards": shards, "codes_per_shard": int(n_per),
            "queries_in_batch": int(queries.shape[0]),
            "sharded_vs_unsharded": {"queries_checked": int(queries.shape[0]), "mismatches": len(shard_bad),
                                     "mismatched_queries": shard_bad[:50]},
            "oracle": {"queries_checked": int(len(sample)), "sample_seed": 20261020,
                       "mismatches": len(bad), "mismatched_queries": bad,
                       "result_ids_per_shard": ids_per_shard,
                       "how": "oracle/pqscan_oracle.py compute_tables + qadc_params over the global 1,000-code "
                              "prefix + quantize, then oracle/qadc_oracle.c quantized_distances + _select_best "
                              "over all 1e9 codes"},
            "compared": "bins and ids", "gpu_phase_s": round(gpu_s, 1), "seconds": round(time.time() - t0, 1)}


def main(argv):
    out = None
    if "--out" in argv:
        k = argv.index("--out")
        out = argv[k + 1]
        argv = argv[:k] + argv[k + 2:]
    names = argv or ["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"]
    report = {"cores": len(os.sched_getaffinity(0)), "results": []}
    for nm in names:
        res = billion() if nm == "cfg4" else ivf() if nm == "cfg3" else exhaustive(nm)
        print(json.dumps(res), flush=True)
        report["results"].append(res)
        if out:
            json.dump(report, open(out, "w"), indent=1)
    return report


if __name__ == "__main__":
    main(sys.argv[1:])
