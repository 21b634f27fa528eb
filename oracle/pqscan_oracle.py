"""CPU oracle for the PQ ADC scan path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference package `pqscan`
(arxiv/paper_1712_02912, `/root/reference/pkg/src/pqscan/`) for exactly the
functions on the hot path.  Every function cites the
reference file:line it follows.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg
(`--impl reference` / `cpu_baseline`) may import this module, and only as the
checker or as the timed CPU baseline.  The product package
(`paper_1712_02912_b200`) never imports it: the product path runs on the GPU
through `libpqs.so` and fails loudly when that library is missing.

Parity pin: `tests/golden/*.npz` were produced by running the real reference
(`tests/golden/make_golden.py`, imported from /root/reference in the build
container); `tests/test_oracle_golden.py` checks this restatement against
every fixture bit-for-bit.

Third-party arithmetic (not vendored in the reference):
  * scipy.spatial.distance.cdist(.., 'sqeuclidean') (scipy>=1.10, unpinned) --
    restated as fp64 direct differences (`_dist.py:13-21`); the golden
    fixtures pin the bitwise fp32 result of `compute_tables`.
  * numpy partition/lexsort/floor/clip/minimum (numpy>=1.24) -- restated with
    the same semantics; ties are pinned by the sorted-oracle fixtures.
"""

from __future__ import annotations

import heapq

import numpy as np

BINS = 127          # fastscan.py:23
BLOCK = 16          # scan.py:206
DEFAULT_INIT_COUNT = 200            # quickadc.py:28
DEFAULT_INIT_COUNT_BILLION = 1000   # quickadc.py:29


# --------------------------------------------------------------------------
# tables  (scan.py:45-56, _dist.py:13-21, quantizer.py:85-89)
# --------------------------------------------------------------------------

def compute_tables(codebooks: np.ndarray, query: np.ndarray) -> np.ndarray:
    """D[j, i] = fp32(sum_t (fp64(y_j[t]) - fp64(C_j[i, t]))^2).

    scan.py:45-56 calls `sqdist_matrix` (_dist.py:13-21, scipy cdist
    'sqeuclidean' in fp64) per sub-space on the fp64-cast query
    (quantizer.py:85-89, identity rotation) and stores the row as fp32.
    """
    codebooks = np.asarray(codebooks, dtype=np.float32)
    m, k, dsub = codebooks.shape
    y = np.asarray(query, dtype=np.float64).reshape(m, 1, dsub)
    diff = y - codebooks.astype(np.float64)
    out = np.zeros((m, k), dtype=np.float64)
    for t in range(dsub):  # scipy cdist 'sqeuclidean': sequential fp64 sum
        out += diff[:, :, t] * diff[:, :, t]
    return out.astype(np.float32)


def compute_tables_batch(codebooks: np.ndarray, queries: np.ndarray) -> np.ndarray:
    """compute_tables for a (Q, d) batch -> (Q, m, k) float32."""
    queries = np.asarray(queries)
    return np.stack([compute_tables(codebooks, q) for q in queries])


# --------------------------------------------------------------------------
# float ADC  (scan.py:59-81)
# --------------------------------------------------------------------------

def adc_distance(tables: np.ndarray, code) -> float:
    """scan.py:59-65: fp64 sum of fp32 entries, sub-space order."""
    acc = 0.0
    for j in range(tables.shape[0]):
        acc += float(tables[j, int(code[j])])
    return acc


def scan_distances(tables: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """scan.py:68-81: acc(fp64) += T64[j][codes[:, j]] for j = 0..m-1."""
    t64 = np.asarray(tables, dtype=np.float32).astype(np.float64)
    codes = np.asarray(codes)
    acc = np.zeros(codes.shape[0], dtype=np.float64)
    for j in range(t64.shape[0]):
        acc += t64[j][codes[:, j].astype(np.int64)]
    return acc


# --------------------------------------------------------------------------
# selection  (scan.py:84-154)
# --------------------------------------------------------------------------

def select_best(dists: np.ndarray, ids: np.ndarray, r: int):
    """scan.py:142-154: the r smallest (distance, id) pairs, ascending."""
    n = dists.shape[0]
    r_eff = min(r, n)
    if r_eff == 0:
        return np.empty(0, np.float64), np.empty(0, np.int64)
    kth = np.partition(dists, r_eff - 1)[r_eff - 1]
    cand = np.flatnonzero(dists <= kth)
    order = np.lexsort((ids[cand], dists[cand]))[:r_eff]
    pick = cand[order]
    return dists[pick], ids[pick]


class NeighborMerge:
    """Bounded (distance, id) set with the NeighborSet.push semantics of
    scan.py:109-118: keeps the r smallest by (distance, id)."""

    def __init__(self, r: int):
        if r < 1:
            raise ValueError("r must be >= 1")
        self.r = r
        self._heap: list = []

    def push(self, distance: float, ident: int) -> bool:
        entry = (-float(distance), -int(ident))
        if len(self._heap) < self.r:
            heapq.heappush(self._heap, entry)
            return True
        if entry > self._heap[0]:
            heapq.heappushpop(self._heap, entry)
            return True
        return False

    def worst(self) -> float:
        """scan.py:102-107: the r-th best distance, inf while fewer are held."""
        return float("inf") if len(self._heap) < self.r else -self._heap[0][0]

    def items(self):
        return sorted((-d, -i) for d, i in self._heap)


def scan(codes: np.ndarray, ids: np.ndarray, tables: np.ndarray, r: int):
    """scan.py:197-203 -> (dists fp64, ids int64) ascending by (d, id)."""
    if r < 1:
        raise ValueError("r must be >= 1")
    d = scan_distances(tables, codes)
    return select_best(d, np.asarray(ids, dtype=np.int64), r)


# --------------------------------------------------------------------------
# 16-code block layout  (scan.py:206-287)
# --------------------------------------------------------------------------

def transpose_blocks(codes: np.ndarray, b: int) -> np.ndarray:
    """scan.py:248-274 -> blocks (nblocks, rows, 16) uint8."""
    codes = np.asarray(codes)
    n, m = codes.shape
    if b == 4:
        if m % 2:
            raise ValueError("b=4 transposition needs even m")
        if np.any(codes >= 16):
            raise ValueError("component out of range for b=4")
    elif b == 8:
        if np.any(codes.astype(np.int64) >= 256):
            raise ValueError("component out of range for b=8")
    else:
        raise ValueError(f"block transposition supports b in (4, 8), got b={b}")
    nblocks = (n + BLOCK - 1) // BLOCK
    padded = np.zeros((nblocks * BLOCK, m), dtype=np.uint8)
    padded[:n] = codes.astype(np.uint8)
    per_block = padded.reshape(nblocks, BLOCK, m)
    if b == 4:
        blocks = (per_block[:, :, 0::2] | (per_block[:, :, 1::2] << 4)).transpose(0, 2, 1)
    else:
        blocks = per_block.transpose(0, 2, 1)
    return np.ascontiguousarray(blocks)


def detranspose_blocks(blocks: np.ndarray, n: int, m: int, b: int) -> np.ndarray:
    """scan.py:277-287 -> codes (n, m) uint8."""
    nblocks = blocks.shape[0]
    if b == 4:
        flat = blocks.transpose(0, 2, 1).reshape(-1, m // 2)
        codes = np.empty((nblocks * BLOCK, m), dtype=np.uint8)
        codes[:, 0::2] = flat & 0x0F
        codes[:, 1::2] = flat >> 4
    else:
        codes = blocks.transpose(0, 2, 1).reshape(-1, m)
    return np.ascontiguousarray(codes[:n])


# --------------------------------------------------------------------------
# 127-bin quantization  (fastscan.py:28-57, quickadc.py:32-141)
# --------------------------------------------------------------------------

def quant_scale(qmin: float, qmax: float) -> float:
    """fastscan.py:42-45."""
    span = qmax - qmin
    return BINS / span if span > 0.0 else 0.0


def quantize(qmin: float, qmax: float, values) -> np.ndarray:
    """fastscan.py:48-57: 127 at or above qmax, else floor-scaled, clamped
    to [0, 126]; all-zero when the span is empty.  fp64 arithmetic."""
    v = np.asarray(values, dtype=np.float64)
    scale = quant_scale(qmin, qmax)
    if scale == 0.0:
        return np.zeros(v.shape, dtype=np.uint8)
    bins = np.clip(np.floor((v - qmin) * scale), 0, BINS - 1)
    return np.where(v >= qmax, BINS, bins).astype(np.uint8)


def qadc_block(block: np.ndarray, qtables: np.ndarray) -> np.ndarray:
    """quickadc.py:66-84: one transposed 16-code block, clamp after each add."""
    block = np.asarray(block, dtype=np.uint8)
    acc = np.zeros(BLOCK, dtype=np.int16)
    for j in range(block.shape[0]):
        row = block[j]
        acc = np.minimum(acc + qtables[2 * j][row & 0x0F], BINS)
        acc = np.minimum(acc + qtables[2 * j + 1][row >> 4], BINS)
    return acc.astype(np.uint8)


def quantized_distances(codes: np.ndarray, qtables: np.ndarray) -> np.ndarray:
    """quickadc.py:87-101: int16 acc = min(acc + t[j][c_j], 127)."""
    codes = np.asarray(codes)
    acc = np.zeros(codes.shape[0], dtype=np.int16)
    for j in range(qtables.shape[0]):
        acc = np.minimum(acc + qtables[j][codes[:, j].astype(np.int64)], BINS)
    return acc.astype(np.uint8)


def qadc_params(tables: np.ndarray, codes: np.ndarray, init_count: int, r: int):
    """quickadc.py:129-137 -> (qmin, qmax) fp64.

    qmax = r-th smallest fp64 ADC distance of the first min(init_count, n)
    codes in storage order (largest if fewer than r); qmin = global fp32
    table minimum; qmax = max(qmax, qmin)."""
    n_init = min(init_count, codes.shape[0])
    prefix_d = scan_distances(tables, codes[:n_init])
    if n_init >= r:
        qmax = float(np.partition(prefix_d, r - 1)[r - 1])
    else:
        qmax = float(prefix_d.max())
    qmin = float(np.asarray(tables, dtype=np.float32).min())
    return qmin, max(qmax, qmin)


def qadc_scan(codes: np.ndarray, ids: np.ndarray, tables: np.ndarray,
              init_count: int, r: int):
    """quickadc.py:104-141 on the detransposed codes.

    Returns (bins float64 ascending, ids int64, qtables uint8 (m,16), qmin, qmax).
    """
    tables = np.asarray(tables, dtype=np.float32)
    if tables.shape[1] != 16:
        raise ValueError("tables do not match the code list shape")
    if tables.shape[0] % 2:
        raise ValueError("quick scan needs even m")
    if init_count < 1:
        raise ValueError("init_count must be >= 1")
    if r < 1:
        raise ValueError("r must be >= 1")
    if codes.shape[0] == 0:
        raise ValueError("empty code list")
    qmin, qmax = qadc_params(tables, codes, init_count, r)
    qt = quantize(qmin, qmax, tables)
    dq = quantized_distances(codes, qt).astype(np.float64)
    best_d, best_i = select_best(dq, np.asarray(ids, dtype=np.int64), r)
    return best_d, best_i, qt, qmin, qmax


def rescale(bins, qmin: float, qmax: float):
    """quickadc.py:50-54."""
    return np.asarray(bins, dtype=np.float64) * (qmax - qmin) / BINS + qmin


# --------------------------------------------------------------------------
# IVFADC  (_dist.py:42-67, ivf.py:148-196)
# --------------------------------------------------------------------------

def sqdist_matrix(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """_dist.py:13-21: fp64 all-pairs squared distances, direct form,
    summed sequentially over t (bit-identical to scipy 1.18 cdist)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    out = np.empty((a.shape[0], b.shape[0]), dtype=np.float64)
    step = max(1, min(64, (1 << 22) // max(1, b.shape[0] * b.shape[1])))  # bounded temporaries
    for lo in range(0, a.shape[0], step):
        d = a[lo:lo + step, None, :] - b[None, :, :]
        acc = np.zeros(d.shape[:2], dtype=np.float64)
        for t in range(d.shape[2]):  # sequential order, as scipy's cdist
            acc += d[:, :, t] * d[:, :, t]
        out[lo:lo + step] = acc
    return out


def nearest_k(points: np.ndarray, centroids: np.ndarray, k: int):
    """_dist.py:42-67: k nearest by (fp64 distance, index), ascending."""
    points = np.atleast_2d(np.asarray(points))
    n = points.shape[0]
    idx = np.empty((n, k), dtype=np.int64)
    dist = np.empty((n, k), dtype=np.float64)
    ncent = centroids.shape[0]
    cent_ids = np.arange(ncent)
    dm_all = sqdist_matrix(points, centroids)
    for row in range(n):
        d = dm_all[row]
        if k < ncent:
            kth = np.partition(d, k - 1)[k - 1]
            cand = np.flatnonzero(d <= kth)
        else:
            cand = cent_ids
        order = np.lexsort((cand, d[cand]))[:k]
        sel = cand[order]
        idx[row] = sel
        dist[row] = d[sel]
    return idx, dist


def encode(codebooks: np.ndarray, x: np.ndarray, coarse: np.ndarray | None = None,
           cells: np.ndarray | None = None) -> np.ndarray:
    """quantizer.py:308-325 (identity rotation -> fp64 rows) with nearest
    (_dist.py:24-39): per sub-space the argmin of the fp64 sequential-sum
    distances, ties to the lowest index.  With coarse/cells: the IVF residual
    fp64(x) - fp64(coarse[cells]) as build_ivf encodes it (ivf.py:137-140)."""
    books = np.asarray(codebooks, dtype=np.float32)
    m, k, dsub = books.shape
    z = np.asarray(x, dtype=np.float64)
    if coarse is not None:
        z = z - np.asarray(coarse, np.float32).astype(np.float64)[np.asarray(cells, np.int64)]
    out = np.empty((z.shape[0], m), dtype=np.uint8 if k <= 256 else np.uint16)
    for j in range(m):
        dm = sqdist_matrix(z[:, j * dsub:(j + 1) * dsub], books[j].astype(np.float64))
        out[:, j] = np.argmin(dm, axis=1)
    return out


def query_ivf(coarse: np.ndarray, codebooks: np.ndarray, lists_codes, lists_ids,
              query: np.ndarray, ma: int, r: int, kernel: str = "adc", init_count: int = 200):
    """ivf.py:148-196, kernels 'adc' and 'quick-adc': probe the ma nearest
    cells, scan each list against the fp64 residual's tables ('adc': exact
    ADC, ivf.py:181-184; 'quick-adc': qadc_scan with min(init_count, n) and
    its bins rescaled, ivf.py:185-190), merge by (distance, id)."""
    K = coarse.shape[0]
    if not 1 <= ma <= K:
        raise ValueError(f"ma must be in [1, {K}]")
    if r < 1:
        raise ValueError("r must be >= 1")
    q64 = np.asarray(query, dtype=np.float64)
    cells, _ = nearest_k(q64[None, :], np.asarray(coarse, np.float32).astype(np.float64), ma)
    merged = NeighborMerge(r)
    for cell in cells[0]:
        codes = lists_codes[int(cell)]
        if codes.shape[0] == 0:
            continue
        residual = q64 - np.asarray(coarse[int(cell)], np.float32).astype(np.float64)
        tables = compute_tables(codebooks, residual)
        if kernel == "quick-adc":
            bins, ids, _, qmin, qmax = qadc_scan(codes, lists_ids[int(cell)], tables,
                                                 min(init_count, codes.shape[0]), r)
            d = rescale(bins, qmin, qmax)
        else:
            d, ids = scan(codes, lists_ids[int(cell)], tables, r)
        for dist, ident in zip(d.tolist(), ids.tolist()):
            merged.push(dist, ident)
    items = merged.items()
    return (np.array([p[0] for p in items], dtype=np.float64),
            np.array([p[1] for p in items], dtype=np.int64))


# --------------------------------------------------------------------------
# sharded merge  (scan.py:109-118 semantics; no reference counterpart)
# --------------------------------------------------------------------------

def merge_shards(dists_list, ids_list, r: int):
    """Top-r of the union of per-shard top-r lists by (distance, id)."""
    d = np.concatenate([np.asarray(x, np.float64) for x in dists_list])
    i = np.concatenate([np.asarray(x, np.int64) for x in ids_list])
    return select_best(d, i, r)


# --------------------------------------------------------------------------
# PQ Fast Scan  (fastscan.py:208-386)
# --------------------------------------------------------------------------

def group_order(codes: np.ndarray) -> np.ndarray:
    """fastscan.py:208-219: stable order by the high nibbles of components 0-3."""
    highs = (np.asarray(codes)[:, :4] >> 4).astype(np.uint32)
    key_val = (highs[:, 0] << 12) | (highs[:, 1] << 8) | (highs[:, 2] << 4) | highs[:, 3]
    return np.argsort(key_val, kind="stable")


def fast_scan(codes: np.ndarray, ids: np.ndarray, tables: np.ndarray, init: float, r: int):
    """fastscan.py:328-386 on codes in grouped storage order: the sequential
    pruned scan.  Returns (dists, ids, checked, pruned)."""
    import math

    tables = np.asarray(tables, dtype=np.float32)
    ids = np.asarray(ids, dtype=np.int64)
    n = codes.shape[0]
    merged = NeighborMerge(r)
    if n == 0:
        return np.empty(0), np.empty(0, np.int64), 0, 0
    n_init = math.ceil(init * n)
    prefix_d = scan_distances(tables, codes[:n_init])
    checked, pruned = n_init, 0
    order = np.lexsort((ids[:n_init], prefix_d))
    for pos in order[: min(r, n_init)]:
        merged.push(float(prefix_d[pos]), int(ids[pos]))
    qmax = float(np.partition(prefix_d, r - 1)[r - 1]) if n_init >= r else float(prefix_d.max())
    qmin = float(tables.min())
    qmax = max(qmax, qmin)
    qt = quantize(qmin, qmax, tables)
    mins = qt[4:8].reshape(4, 16, 16).min(axis=2)                 # fastscan.py:258-260
    start = n_init
    while start < n:
        stop = min(start + 1024, n)
        chunk = codes[start:stop]
        worst = merged.worst()
        threshold = int(quantize(qmin, qmax, np.array([worst]))[0])
        idx = chunk.astype(np.int64)                               # _lower_bounds_all, fastscan.py:300-310
        acc = qt[0][idx[:, 0]].astype(np.int16)
        for j in range(1, 4):
            acc += qt[j][idx[:, j]]
        for j in range(4, 8):
            acc += mins[j - 4][idx[:, j] >> 4]
        lb = np.minimum(acc, BINS)
        keep = lb <= threshold
        pruned += int(np.count_nonzero(~keep))
        kept = np.flatnonzero(keep)
        if kept.size:
            d = scan_distances(tables, chunk[kept])
            checked += kept.size
            kid = ids[start:stop][kept]
            for pos in np.lexsort((kid, d)):
                if not merged.push(float(d[pos]), int(kid[pos])):
                    break
        start = stop
    items = merged.items()
    return (np.array([p[0] for p in items], dtype=np.float64), np.array([p[1] for p in items], dtype=np.int64),
            checked, pruned)


# --------------------------------------------------------------------------
# Derived quantizers: two-pass search  (derived.py:129-409)
# --------------------------------------------------------------------------

def quantize_255(qmin: float, qmax: float, values) -> np.ndarray:
    """derived.py:143-154."""
    v = np.asarray(values, dtype=np.float64)
    span = qmax - qmin
    if span <= 0.0:
        return np.zeros(v.shape, dtype=np.uint8)
    bins = np.clip(np.floor((v - qmin) * (255 / span)), 0, 254)
    return np.where(v >= qmax, 255, bins).astype(np.uint8)


def search_two_pass(full_books: np.ndarray, derived_books: np.ndarray, codes: np.ndarray, ids: np.ndarray,
                    query: np.ndarray, r: int, r2: int):
    """derived.py:402-409 restated: compact tables (129-140), 255-bin
    quantization with qmax = max ADC of the first min(r2, n) codes' low bits
    (180-198), the admission rule of scan_candidates (294-326) and the exact
    rerank of the admitted codes (362-399)."""
    codes = np.asarray(codes)
    ids = np.asarray(ids, dtype=np.int64)
    n = codes.shape[0]
    if n == 0:
        raise ValueError("empty code list")
    kbar = derived_books.shape[1]
    compact = compute_tables(derived_books, query)
    low = (codes.astype(np.int64) & (kbar - 1))
    qmin = float(compact.min())
    qmax = max(float(scan_distances(compact, low[: min(r2, n)]).max()), qmin)
    qt = quantize_255(qmin, qmax, compact)
    acc = np.zeros(n, dtype=np.int32)
    for j in range(qt.shape[0]):
        acc = np.minimum(acc + qt[j][low[:, j]], 255)
    d = acc.astype(np.uint8)
    smalls = d <= 254
    if int(np.count_nonzero(smalls)) >= r2:
        hist = np.bincount(d[smalls], minlength=255)
        bound = int(np.argmax(np.cumsum(hist) >= r2))
        sel = d <= bound
    else:
        # put() in storage order: a d = 255 code is admitted while fewer than
        # r2 are held (scan_candidates, derived.py:316-323)
        sel = smalls.copy()
        held = 0
        for p in range(n):
            if smalls[p]:
                held += 1
            elif held < r2:
                sel[p] = True
                held += 1
    pick = np.flatnonzero(sel)
    full = compute_tables(full_books, query)
    dist = scan_distances(full, codes[pick])
    return select_best(dist, ids[pick], r)


def query_ivf_derived(coarse, full_books, derived_books, lists_codes, lists_ids, query, ma: int, r: int, r2: int):
    """ivf.py:148-196 with kernel='derived' (191-195)."""
    q64 = np.asarray(query, dtype=np.float64)
    cells, _ = nearest_k(q64[None, :], np.asarray(coarse, np.float32).astype(np.float64), ma)
    merged = NeighborMerge(r)
    for cell in cells[0]:
        codes = lists_codes[int(cell)]
        if codes.shape[0] == 0:
            continue
        residual = q64 - np.asarray(coarse[int(cell)], np.float32).astype(np.float64)
        d, ids = search_two_pass(full_books, derived_books, codes, lists_ids[int(cell)], residual, r, r2)
        for dist, ident in zip(d.tolist(), ids.tolist()):
            merged.push(dist, ident)
    items = merged.items()
    return (np.array([p[0] for p in items], dtype=np.float64), np.array([p[1] for p in items], dtype=np.int64))
