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

from ._cache import device_cached
from .engine import DeviceCodes, DeviceQuantizer
from .types import BLOCK, CodeList, LookupTables, NeighborSet, ProductQuantizer, TransposedCodeList, implicit_ids


def _device_quantizer(pq: ProductQuantizer) -> DeviceQuantizer:
    return device_cached(pq, "_pqs_dev", (pq.codebooks, pq.rotation), lambda: DeviceQuantizer(pq))


def _device_codes(obj, source: np.ndarray, b: int, convert=None) -> DeviceCodes:
    """Device copy of obj's codes (source: the container's own array, frozen;
    convert: source -> (n, m) uint8 codes) with obj's ids (implicit while
    they are the container's default arange)."""
    ids = None if implicit_ids(obj) else obj.ids
    return device_cached(obj, f"_pqs_dev{b}", (source, obj.ids),
                         lambda: DeviceCodes(convert(source) if convert else source, b, ids=ids))


def compute_tables(pq: ProductQuantizer, query: np.ndarray) -> LookupTables:
    """scan.py:45-56 -- squared distances from each query sub-vector to every centroid."""
    query = np.asarray(query)
    if query.ndim != 1 or query.shape[0] != pq.d:
        raise ValueError(f"query must have shape ({pq.d},)")
    dq = _device_quantizer(pq)
    return LookupTables(dq.compute_tables(query[None, :])[0])


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
    codes = codelist.codes
    if codes.size and int(codes.max()) >= max(tables.k, 1):
        raise IndexError("code component out of range for the tables")
    dev = _device_codes(codelist, codes, 8, lambda c: _codes_u8(c, tables.k))
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
    object.__setattr__(out, "_implicit_ids", codelist.__dict__.get("_implicit_ids"))
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
