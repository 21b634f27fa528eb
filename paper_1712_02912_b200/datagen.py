"""Seeded synthetic stand-ins for the BASELINE.json configs (data prep only).

The reference measures on SIFT1M / GIST1M / Deep1B-style corpora that are not
in this environment; these generators reproduce the configs' shapes and value
distributions (BASELINE.json `configs`), deterministically from fixed seeds
(numpy PCG64, one generator per 65,536-row chunk so any chunk can be rebuilt
alone).  Codebooks are trained with plain Lloyd k-means (random init, fp32
matmul distances) -- quantizer training is outside the scan path;
the scan, its parity and its timing do not depend on how the codebooks were
trained.
"""

from __future__ import annotations

import numpy as np

CHUNK = 1 << 16


def _mixture_centers(seed: int, comps: int, d: int, hi: float) -> np.ndarray:
    return np.random.default_rng([seed, 0xC0]).uniform(0.0, hi, size=(comps, d))


def mixture_rows(seed: int, lo: int, hi_row: int, d: int, comps: int, center_hi: float, sigma: float,
                 clip_lo: float | None, clip_hi: float | None, stream: int = 0) -> np.ndarray:
    """Rows [lo, hi_row) of a seeded isotropic Gaussian mixture (float32)."""
    centers = _mixture_centers(seed, comps, d, center_hi)
    out = np.empty((hi_row - lo, d), dtype=np.float32)
    for c0 in range((lo // CHUNK) * CHUNK, hi_row, CHUNK):
        rng = np.random.default_rng([seed, stream, c0 // CHUNK])
        n = CHUNK
        lab = rng.integers(0, comps, size=n)
        x = centers[lab] + rng.normal(0.0, sigma, size=(n, d))
        if clip_lo is not None or clip_hi is not None:
            x = np.clip(x, clip_lo, clip_hi)
        a, b = max(lo, c0), min(hi_row, c0 + CHUNK)
        out[a - lo:b - lo] = x[a - c0:b - c0]
    return out


def decay_gaussian_rows(seed: int, lo: int, hi_row: int, d: int = 96, stream: int = 0) -> np.ndarray:
    """cfg4: per-dimension variance 1/(1+i), then L2-normalised (float32)."""
    std = 1.0 / np.sqrt(1.0 + np.arange(d))
    out = np.empty((hi_row - lo, d), dtype=np.float32)
    for c0 in range((lo // CHUNK) * CHUNK, hi_row, CHUNK):
        rng = np.random.default_rng([seed, stream, c0 // CHUNK])
        x = rng.normal(0.0, 1.0, size=(CHUNK, d)) * std
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        a, b = max(lo, c0), min(hi_row, c0 + CHUNK)
        out[a - lo:b - lo] = x[a - c0:b - c0]
    return out


CONFIGS = {
    # name: generator kwargs, d, m, b, N, Q (BASELINE.json configs[0..4])
    "cfg0": dict(kind="mix", d=128, comps=256, center_hi=128.0, sigma=16.0, clip=(0.0, 255.0), m=8, b=8,
                 N=1_000_000, Q=1000, r=100),
    "cfg1": dict(kind="mix", d=128, comps=256, center_hi=128.0, sigma=16.0, clip=(0.0, 255.0), m=16, b=4,
                 N=1_000_000, Q=1000, r=100, init_count=200),
    "cfg2": dict(kind="mix", d=960, comps=64, center_hi=1.0, sigma=0.05, clip=(0.0, None), m=64, b=8,
                 N=1_000_000, Q=1000, r=100),
    "cfg3": dict(kind="mix", d=128, comps=256, center_hi=128.0, sigma=16.0, clip=(0.0, 255.0), m=8, b=8,
                 N=100_000_000, Q=10_000, r=100, K=65536, nprobe=64),
    "cfg4": dict(kind="decay", d=96, m=16, b=4, N=1_000_000_000, Q=10_000, r=100, init_count=1000),
}


def rows(cfg: dict, seed: int, lo: int, hi_row: int, stream: int = 0) -> np.ndarray:
    """Rows [lo, hi_row); chunks are generated in parallel (each has its own seed)."""
    from concurrent.futures import ThreadPoolExecutor

    step = CHUNK * 4
    parts = [(a, min(a + step, hi_row)) for a in range(lo, hi_row, step)]

    def one(ab):
        a, b = ab
        if cfg["kind"] == "mix":
            cl = cfg["clip"]
            return mixture_rows(seed, a, b, cfg["d"], cfg["comps"], cfg["center_hi"], cfg["sigma"], cl[0], cl[1],
                                stream)
        return decay_gaussian_rows(seed, a, b, cfg["d"], stream)

    if len(parts) <= 1:
        return one((lo, hi_row))
    with ThreadPoolExecutor(max_workers=8) as ex:
        return np.concatenate(list(ex.map(one, parts)))


def kmeans(x: np.ndarray, k: int, iters: int, seed: int) -> np.ndarray:
    """Plain Lloyd k-means, random init (fp32 matmul assignment)."""
    rng = np.random.default_rng(seed)
    x = np.ascontiguousarray(x, dtype=np.float32)
    c = x[rng.choice(x.shape[0], k, replace=False)].copy()
    xx = (x * x).sum(1)
    for _ in range(iters):
        dd = (c * c).sum(1)[None] - 2.0 * (x @ c.T)
        a = dd.argmin(1)
        order = np.argsort(a, kind="stable")
        cnt = np.bincount(a, minlength=k)
        nz = np.flatnonzero(cnt)
        starts = np.concatenate([[0], np.cumsum(cnt)[:-1]])[nz]
        sums = np.add.reduceat(x[order].astype(np.float64), starts, axis=0)
        c[nz] = (sums / cnt[nz, None]).astype(np.float32)
    return c


def train_pq(x: np.ndarray, m: int, b: int, iters: int = 20, seed: int = 0) -> np.ndarray:
    from concurrent.futures import ThreadPoolExecutor

    d = x.shape[1]
    dsub = d // m
    k = 1 << b
    with ThreadPoolExecutor(max_workers=min(m, 16)) as ex:
        books = list(ex.map(lambda j: kmeans(x[:, j * dsub:(j + 1) * dsub], k, iters, seed + j), range(m)))
    return np.stack(books)


def encode(books: np.ndarray, x: np.ndarray, chunk: int = 1 << 16) -> np.ndarray:
    """Nearest centroid per sub-space (fp32 matmul expansion; data prep only)."""
    from concurrent.futures import ThreadPoolExecutor

    m, k, dsub = books.shape
    out = np.empty((x.shape[0], m), dtype=np.uint8)
    cn = (books * books).sum(2)

    def work(lo):
        xs = x[lo:lo + chunk]
        for j in range(m):
            sub = xs[:, j * dsub:(j + 1) * dsub]
            dd = cn[j][None] - 2.0 * (sub @ books[j].T)
            out[lo:lo + chunk, j] = dd.argmin(1)

    with ThreadPoolExecutor(max_workers=8) as ex:
        list(ex.map(work, range(0, x.shape[0], chunk)))
    return out


def make_exhaustive(name: str, seed: int = 1712, n: int | None = None, nq: int | None = None,
                    shard: int = 0, train_rows: int = 100_000):
    """(codebooks, codes, queries) for cfg0/1/2 (and shard-local cfg1-style data)."""
    cfg = CONFIGS[name]
    n = cfg["N"] if n is None else n
    nq = cfg["Q"] if nq is None else nq
    train = rows(cfg, seed, 0, train_rows, stream=0)
    books = train_pq(train, cfg["m"], cfg["b"], iters=20, seed=seed)
    base = rows(cfg, seed, shard * n, (shard + 1) * n, stream=1)
    codes = encode(books, base)
    queries = rows(cfg, seed, 0, nq, stream=2)
    return books, codes, queries
