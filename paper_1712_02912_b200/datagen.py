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


# ------------------------------------------------------------------ device
# cfg3 / cfg4 are too large to generate on the host (1e8 x 128 and 1e9 x 96
# float32): rows are drawn on the GPU with torch's counter-based Philox
# generator, one generator per 2^20-row chunk keyed by (seed, stream, chunk)
# (SURVEY 8d), same distributions as the host generators above.
DCHUNK = 1 << 20


def _chunk_seed(seed: int, stream: int, chunk: int) -> int:
    return int(np.random.SeedSequence([seed, stream, chunk, 0xD7]).generate_state(1, np.uint64)[0] >> 1)


def device_rows(cfg: dict, seed: int, lo: int, hi_row: int, stream: int = 0, device="cuda"):
    """Rows [lo, hi_row) as a float32 CUDA tensor (chunks rebuilt independently)."""
    import torch

    d = cfg["d"]
    out = torch.empty((hi_row - lo, d), dtype=torch.float32, device=device)
    if cfg["kind"] == "mix":
        centers = torch.from_numpy(_mixture_centers(seed, cfg["comps"], d, cfg["center_hi"]).astype(np.float32)).to(
            device)
    else:
        std = torch.from_numpy((1.0 / np.sqrt(1.0 + np.arange(d))).astype(np.float32)).to(device)
    for c in range(lo // DCHUNK, (hi_row + DCHUNK - 1) // DCHUNK):
        g = torch.Generator(device=device)
        g.manual_seed(_chunk_seed(seed, stream, c))
        c0 = c * DCHUNK
        if cfg["kind"] == "mix":
            lab = torch.randint(0, cfg["comps"], (DCHUNK,), generator=g, device=device)
            x = centers[lab] + torch.randn((DCHUNK, d), generator=g, device=device) * cfg["sigma"]
            lo_c, hi_c = cfg["clip"]
            x = x.clamp(min=lo_c, max=hi_c)
        else:
            x = torch.randn((DCHUNK, d), generator=g, device=device) * std
            x = x / x.norm(dim=1, keepdim=True)
        a, b = max(lo, c0), min(hi_row, c0 + DCHUNK)
        out[a - lo:b - lo] = x[a - c0:b - c0]
    return out


def device_encode_rows(dq, cfg: dict, seed: int, lo: int, hi_row: int, stream: int = 1, device="cuda",
                       chunk: int = 1 << 22):
    """Codes of rows [lo, hi_row) generated and encoded on the GPU (exact
    encode kernel, quantizer.py:308-325); returns a (n, m) uint8 CUDA tensor."""
    import torch

    n = hi_row - lo
    codes = torch.empty((n, cfg["m"]), dtype=torch.uint8, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        codes[a:b] = dq.encode(device_rows(cfg, seed, lo + a, lo + b, stream, device))
    return codes


def make_quick_adc_shard(name: str, rank: int, world: int, dq_factory, seed: int = 1712, n: int | None = None,
                         nq: int | None = None, train_rows: int = 100_000, device="cuda"):
    """cfg4-style shard on the device: (books, codes (n, m) CUDA uint8 of global
    rows [rank*n, (rank+1)*n), prefix codes (init_count, m) of global rows
    [0, init_count), host queries).  dq_factory(books) -> DeviceQuantizer."""
    cfg = CONFIGS[name]
    n = cfg["N"] // world if n is None else n
    nq = cfg["Q"] if nq is None else nq
    train = rows(cfg, seed, 0, train_rows, stream=0)
    books = train_pq(train, cfg["m"], cfg["b"], iters=20, seed=seed)
    dq = dq_factory(books)
    codes = device_encode_rows(dq, cfg, seed, rank * n, (rank + 1) * n, stream=1, device=device)
    prefix = device_encode_rows(dq, cfg, seed, 0, cfg["init_count"], stream=1, device=device)
    queries = rows(cfg, seed, 0, nq, stream=2)
    return books, codes, prefix, queries


def kmeans_device(x, k: int, iters: int, seed: int, chunk: int = 8192):
    """Lloyd k-means on the GPU for the coarse quantizer (data prep only --
    training is outside the scan path; TF32 matmul assignment)."""
    import torch

    g = torch.Generator(device=x.device)
    g.manual_seed(seed)
    c = x[torch.randperm(x.shape[0], generator=g, device=x.device)[:k]].clone()
    for _ in range(iters):
        a = assign_device(x, c, chunk)
        sums = torch.zeros_like(c, dtype=torch.float64).index_add_(0, a, x.double())
        cnt = torch.bincount(a, minlength=k)
        nz = cnt > 0
        c[nz] = (sums[nz] / cnt[nz, None]).float()
    return c


def assign_device(x, c, chunk: int = 8192):
    """Nearest centroid per row by ||c||^2 - 2<x, c> with a TF32 GEMM: only the
    Lloyd iterations of the coarse k-means (training, out of scope) use it;
    the index build's assignment is the exact `nearest` (pqs_nearest)."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        cn = (c * c).sum(1)
        out = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
        for a in range(0, x.shape[0], chunk):
            xs = x[a:a + chunk]
            out[a:a + chunk] = torch.addmm(cn[None, :], xs, c.t(), beta=1.0, alpha=-2.0).argmin(1)
        return out
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def make_ivf_device(name: str, dq_factory, seed: int = 1712, n: int | None = None, K: int | None = None,
                    nq: int | None = None, coarse_iters: int = 8, device="cuda", chunk: int = 1 << 22):
    """cfg3-style IVFADC index built on the GPU:
    coarse k-means on a device sample, exact assignment of every row
    (nearest, _dist.py:24-39 / ivf.py:122: pqs_nearest = tcgen05 tf32 probe
    GEMM shortlist + fp64 re-score, ties to the lowest index), residual
    PQ trained on the host from a residual sample (ivf.py:120-134 recipe),
    exact residual encode on the device (encode kernel), lists in cell order
    (stable, ids ascending inside a list as build_ivf's flatnonzero).
    Returns (books, coarse CUDA (K, d), list_sizes host (K,), codes CUDA (n, m),
    ids CUDA (n,), host queries)."""
    import torch

    from .engine import nearest

    cfg = CONFIGS[name]
    n = cfg["N"] if n is None else n
    K = cfg["K"] if K is None else K
    nq = cfg["Q"] if nq is None else nq
    # coarse quantizer: k-means on a sample (20 rows per centroid, >= 1M rows)
    ns = min(n, max(20 * K, 1 << 20))
    coarse = kmeans_device(device_rows(cfg, seed, 0, ns, stream=3, device=device), K, coarse_iters, seed)
    # assignment of every base row (stream 1 = the base vectors)
    cells = torch.empty(n, dtype=torch.int64, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        cells[a:b] = nearest(device_rows(cfg, seed, a, b, stream=1, device=device), coarse)[0]
    # residual PQ from a residual sample (100 * 2^b rows, as build_ivf)
    nt = min(n, 100 * (1 << cfg["b"]))
    xt = device_rows(cfg, seed, 0, nt, stream=1, device=device)
    res = (xt.double() - coarse[cells[:nt]].double()).float().cpu().numpy()
    books = train_pq(res, cfg["m"], cfg["b"], iters=20, seed=seed)
    dq = dq_factory(books)
    codes = torch.empty((n, cfg["m"]), dtype=torch.uint8, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        codes[a:b] = dq.encode(device_rows(cfg, seed, a, b, stream=1, device=device), coarse=coarse,
                               cells=cells[a:b])
    ids = torch.argsort(cells, stable=True)
    codes = codes[ids]
    sizes = torch.bincount(cells, minlength=K).cpu().numpy().astype(np.int64)
    queries = rows(cfg, seed, 0, nq, stream=2)
    return books, coarse, sizes, codes, ids, queries
