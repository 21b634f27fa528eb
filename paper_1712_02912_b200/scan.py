"""Drop-in for `pqscan.scan` (scan.py) on the GPU.

compute_tables / scan_distances / scan run on the device through libpqs.so
(K1 exact tables, K3 float scan + K6 exact fp64 rerank + K5 select).  Results
are bit-identical to the reference: tables are fp64 direct differences summed
sequentially (scipy's cdist order) and rounded to fp32; distances are fp64
sums of the fp32 entries in sub-space order; selection is by (distance, id).
transpose_blocks / detranspose_blocks produce the reference's host container
layout (the device's own code layouts are built by kernels at upload).
"""

from __future__ import annotations

import numpy as np

from .engine import DeviceCodes, DeviceQuantizer
from .types import BLOCK, CodeList, LookupTables, NeighborSet, ProductQuantizer, TransposedCodeList


def _device_quantizer(pq: ProductQuantizer) -> DeviceQuantizer:
    key = (pq.codebooks.ctypes.data, pq.codebooks.shape)
    cache = getattr(pq, "_pqs_dev", None)
    if cache is None or cache[0] != key:
        cache = (key, DeviceQuantizer(pq))
        object.__setattr__(pq, "_pqs_dev", cache)
    return cache[1]


def _device_codes(obj, codes: np.ndarray, ids: np.ndarray | None, b: int) -> DeviceCodes:
    key = (codes.ctypes.data, codes.shape, None if ids is None else (ids.ctypes.data, ids.shape), b)
    cache = getattr(obj, "_pqs_dev", None)
    if cache is None or cache[0] != key:
        cache = (key, DeviceCodes(codes, b, ids=ids))
        object.__setattr__(obj, "_pqs_dev", cache)
    return cache[1]


def compute_tables(pq: ProductQuantizer, query: np.ndarray) -> LookupTables:
    """scan.py:45-56 -- squared distances from each query sub-vector to every centroid."""
    query = np.asarray(query)
    if query.ndim != 1 or query.shape[0] != pq.d:
        raise ValueError(f"query must have shape ({pq.d},)")
    dq = _device_quantizer(pq)
    from .quantizer import as_f32_exact

    return LookupTables(dq.compute_tables(as_f32_exact(query, "compute_tables")[None, :])[0])


def compute_tables_batch(pq: ProductQuantizer, queries: np.ndarray) -> np.ndarray:
    """Batched compute_tables: (nq, d) -> (nq, m, k) float32."""
    return _device_quantizer(pq).compute_tables(queries)


def _codes_u8(codes: np.ndarray, k: int) -> np.ndarray:
    codes = np.asarray(codes)
    if codes.size and int(codes.max()) >= max(k, 1):
        raise IndexError("code component out of range for the tables")
    if k > 256:
        raise NotImplementedError("device tables support k <= 256")
    return np.ascontiguousarray(codes, dtype=np.uint8)


def scan_distances(tables: LookupTables, codes: np.ndarray) -> np.ndarray:
    """scan.py:68-81 -- fp64 ADC of every row, sub-space order, bit-exact."""
    codes = np.asarray(codes)
    if codes.ndim != 2 or codes.shape[1] != tables.m:
        raise ValueError(f"codes must have shape (n, {tables.m})")
    if codes.shape[0] == 0:
        return np.zeros(0, dtype=np.float64)
    dev = DeviceCodes(_codes_u8(codes, tables.k), 8)
    return dev.scan_distances(tables.tables[None])[0]


def adc_distance(tables: LookupTables, code: np.ndarray) -> float:
    """scan.py:59-65 -- the scalar form (one code)."""
    code = np.asarray(code).reshape(1, -1)
    return float(scan_distances(tables, code)[0])


def scan(codelist: CodeList, tables: LookupTables, r: int) -> NeighborSet:
    """scan.py:197-203 -- exhaustive scan: the r best codes by (distance, id)."""
    if r < 1:
        raise ValueError("r must be >= 1")
    if codelist.m != tables.m:
        raise ValueError(f"codes must have shape (n, {tables.m})")
    if codelist.n == 0:
        return NeighborSet(r)
    codes = _codes_u8(codelist.codes, tables.k)
    ids = None if getattr(codelist, "_implicit_ids", False) else codelist.ids
    dev = _device_codes(codelist, codes, ids, 8)
    r_dev = min(r, codelist.n)
    d, i, c = dev.adc_scan(tables.tables[None], r_dev)
    n = int(c[0])
    return NeighborSet.from_pairs(r, d[0, :n], i[0, :n])


def transpose_blocks(codelist: CodeList, b: int) -> TransposedCodeList:
    """scan.py:248-274 -- the reference's 16-code component-major host layout."""
    codes = codelist.codes
    n, m = codes.shape
    if b == 4:
        if m % 2 != 0:
            raise ValueError("b=4 transposition needs even m")
        if np.any(codes >= 16):
            raise ValueError("component out of range for b=4")
        rows = m // 2
    elif b == 8:
        if np.any(codes.astype(np.int64) >= 256):
            raise ValueError("component out of range for b=8")
        rows = m
    else:
        raise ValueError(f"block transposition supports b in (4, 8), got b={b}")
    nblocks = (n + BLOCK - 1) // BLOCK
    padded = np.zeros((nblocks * BLOCK, m), dtype=np.uint8)
    padded[:n] = codes.astype(np.uint8)
    per_block = padded.reshape(nblocks, BLOCK, m)
    if b == 4:
        blocks = np.ascontiguousarray((per_block[:, :, 0::2] | (per_block[:, :, 1::2] << 4)).transpose(0, 2, 1))
    else:
        blocks = np.ascontiguousarray(per_block.transpose(0, 2, 1))
    del rows
    out = TransposedCodeList(blocks=blocks, n=n, m=m, b=b, ids=codelist.ids)
    object.__setattr__(out, "_implicit_ids", getattr(codelist, "_implicit_ids", False))
    return out


def detranspose_blocks(tlist: TransposedCodeList) -> CodeList:
    """scan.py:277-287 -- inverse of transpose_blocks."""
    n, m, b = tlist.n, tlist.m, tlist.b
    if b == 4:
        flat = tlist.blocks.transpose(0, 2, 1).reshape(-1, m // 2)
        codes = np.empty((tlist.n_blocks * BLOCK, m), dtype=np.uint8)
        codes[:, 0::2] = flat & 0x0F
        codes[:, 1::2] = flat >> 4
    else:
        codes = tlist.blocks.transpose(0, 2, 1).reshape(-1, m)
    return CodeList(np.ascontiguousarray(codes[:n]), tlist.ids)
