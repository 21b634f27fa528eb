"""Drop-in for `pqscan.quickadc` (quickadc.py) and `fastscan.quantize` on the GPU.

qadc_scan runs K9 (per-query fp64 quantization parameters from the init
prefix, quantized tables), K4 (PRMT register-LUT scan over 4-code quads,
saturating at 127) and K5 (exact (bin, id) top-r) in libpqs.so.  Bins, ids,
quantized tables and (qmin, qmax) are bit-identical to the reference.
"""

from __future__ import annotations

import numpy as np

from .engine import DeviceCodes, quantize_device
from .scan import _device_codes, detranspose_blocks
from .types import (
    BINS,
    BLOCK,
    DEFAULT_INIT_COUNT,
    DEFAULT_INIT_COUNT_BILLION,
    CodeList,
    LookupTables,
    NeighborSet,
    QuantizedTables4,
    QuantParams,
    TransposedCodeList,
)


def quantize(params: QuantParams, values):
    """fastscan.py:48-57 -- 127 at or above qmax, else floor-scaled, clamped."""
    v = np.asarray(values, dtype=np.float64)
    out = quantize_device(params.qmin, params.qmax, v)
    return int(out[()]) if out.ndim == 0 else out


def quantize_tables_4bit(tables: LookupTables, params: QuantParams) -> QuantizedTables4:
    """quickadc.py:57-63."""
    if tables.k != 16:
        raise ValueError("4-bit tables must have 16 entries per sub-space")
    return QuantizedTables4(quantize(params, tables.tables), params)


def quantized_distances(codes: np.ndarray, qt: QuantizedTables4) -> np.ndarray:
    """quickadc.py:87-101 -- per-code saturating table sums (min(sum, 127))."""
    codes = np.asarray(codes)
    t = qt.tables
    if codes.ndim != 2 or codes.shape[1] != t.shape[0]:
        raise ValueError(f"codes must have shape (n, {t.shape[0]})")
    if codes.shape[0] == 0:
        return np.zeros(0, dtype=np.uint8)
    if t.shape[0] % 2:
        # odd m: pad one zero component (adds 0 to every sum)
        codes = np.concatenate([codes, np.zeros((codes.shape[0], 1), codes.dtype)], axis=1)
        t = np.concatenate([t, np.zeros((1, 16), np.uint8)])
    if np.any(codes >= 16):
        raise IndexError("component out of range for 16-entry tables")
    dev = DeviceCodes(np.ascontiguousarray(codes, dtype=np.uint8), 4)
    return dev.quantized_distances(t[None])[0]


def qadc_block(block: np.ndarray, qt: QuantizedTables4) -> np.ndarray:
    """quickadc.py:66-84 -- distances of one transposed block of 16 codes."""
    block = np.asarray(block, dtype=np.uint8)
    t = qt.tables
    if t.shape[0] % 2 != 0:
        raise ValueError("block kernel needs even m")
    if block.shape != (t.shape[0] // 2, BLOCK):
        raise ValueError(f"block must have shape ({t.shape[0] // 2}, {BLOCK})")
    codes = np.empty((BLOCK, t.shape[0]), dtype=np.uint8)
    codes[:, 0::2] = (block & 0x0F).T
    codes[:, 1::2] = (block >> 4).T
    return quantized_distances(codes, qt)


def qadc_scan(tlist: TransposedCodeList, tables: LookupTables, init_count: int, r: int):
    """quickadc.py:104-141 -- quantized scan; returns (NeighborSet of bins, QuantizedTables4)."""
    if tlist.b != 4:
        raise ValueError("quick scan requires 4-bit codes")
    if tables.k != 16 or tables.m != tlist.m:
        raise ValueError("tables do not match the code list shape")
    if tlist.m % 2 != 0:
        raise ValueError("quick scan needs even m")
    if init_count < 1:
        raise ValueError("init_count must be >= 1")
    if r < 1:
        raise ValueError("r must be >= 1")
    if tlist.n == 0:
        raise ValueError("empty code list")
    dev = _device_codes(tlist, tlist.blocks, 4, lambda _: detranspose_blocks(tlist).codes)
    r_dev = min(r, tlist.n)
    bins, oid, cnt, qt, qmm = dev.qadc_scan(tables.tables[None], int(init_count), r_dev)
    n = int(cnt[0])
    params = QuantParams(qmin=float(qmm[0, 0]), qmax=float(qmm[0, 1]))
    nset = NeighborSet.from_pairs(r, bins[0, :n].astype(np.float64), oid[0, :n])
    return nset, QuantizedTables4(qt[0], params)


__all__ = [
    "BINS", "DEFAULT_INIT_COUNT", "DEFAULT_INIT_COUNT_BILLION", "QuantizedTables4", "QuantParams",
    "quantize", "quantize_tables_4bit", "quantized_distances", "qadc_block", "qadc_scan", "CodeList",
]
