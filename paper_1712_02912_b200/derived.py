"""Drop-in for the search side of `pqscan.derived` (derived.py:35-449),
SURVEY 8f row 4: derived low-resolution quantizers sharing codes with the
full ones, and the two-pass search.

`search_two_pass` runs on the device (derived.cu): exact full and compact
tables (K1), 255-bin compact tables, the histogram of the saturated
low-bit sums, the reference's candidate-admission rule (scan_candidates),
and an exact fp64 re-score + (distance, id) selection of every kept code
(rerank) -- results identical to the reference.  `query_ivf(kernel=
'derived')` runs it per probed list (ivf.py:191-195).  Training
(build_derived_quantizers / train_derived: same-size k-means) is out of
scope; DerivedPQ files (PQZ1 + bbar + derived codebooks) and IVF1 files with
a derived quantizer load and save byte-compatibly.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import BinaryIO

import numpy as np

from ._lib import ptr
from .engine import DeviceCodes, DeviceQuantizer, _empty, _fn, _io, _queries
from .formats import _read_array, _read_i32, _write_array, _write_i32, read_quantizer_body, write_quantizer_body
from ._cache import device_cached
from .types import CodeList, LookupTables, NeighborSet, ProductQuantizer, _Sealable, implicit_ids

CBINS = 255  # derived.py:31


@dataclass
class DerivedPQ(_Sealable):
    """derived.py:35-62: full b-bit quantizer + per-sub-space 2^bbar derived
    codebooks; the low bbar bits of a full index name its derived cluster."""

    pq: ProductQuantizer
    bbar: int
    derived: np.ndarray

    def __post_init__(self):
        if not 1 <= self.bbar <= self.pq.b:
            raise ValueError(f"bbar={self.bbar} out of range [1, {self.pq.b}]")
        self.derived = np.ascontiguousarray(self.derived, dtype=np.float32)
        expect = (self.pq.m, 1 << self.bbar, self.pq.dsub)
        if self.derived.shape != expect:
            raise ValueError(f"derived shape {self.derived.shape}, expected {expect}")
        self._seal()

    @property
    def kbar(self) -> int:
        return 1 << self.bbar

    def low_bits(self, indexes):
        out = np.asarray(indexes, dtype=np.int64) & (self.kbar - 1)
        return int(out[()]) if out.ndim == 0 else out

    def _device(self):
        """(full, derived) device quantizer handles, cached on the object."""
        def build():
            dq = ProductQuantizer(m=self.pq.m, b=self.bbar, d=self.pq.d, codebooks=self.derived)
            return DeviceQuantizer(self.pq), DeviceQuantizer(dq)

        return device_cached(self, "_pqs_dev", (self.pq.codebooks, self.derived, self.bbar), build)


def compute_compact_tables(dpq: DerivedPQ, query: np.ndarray) -> LookupTables:
    """derived.py:129-140: squared distances to the derived centroids (K1)."""
    query = np.asarray(query)
    if query.ndim != 1 or query.shape[0] != dpq.pq.d:
        raise ValueError(f"query must have shape ({dpq.pq.d},)")
    _, dd = dpq._device()
    return LookupTables(dd.compute_tables(query[None, :])[0])


def _device_list(db: CodeList) -> DeviceCodes:
    ids = None if implicit_ids(db) else db.ids
    return device_cached(db, "_pqs_dv", (db.codes, db.ids),
                         lambda: DeviceCodes(np.ascontiguousarray(db.codes, dtype=np.uint8), 8, ids=ids))


def search_two_pass_batch(dpq: DerivedPQ, db: CodeList, queries, r: int, r2: int):
    """Batched search_two_pass: (nq, d) -> (dist (nq, r), ids (nq, r), count (nq,))."""
    if db.n == 0:
        raise ValueError("empty code list")              # quantize_compact_tables, derived.py:147-148
    if r2 < 1:
        raise ValueError("r2 must be >= 1")
    if r < 1:
        raise ValueError("r must be >= 1")
    full, dd = dpq._device()
    dev = _device_list(db)
    q, f64 = _queries(queries, 2, "queries")
    nq = q.shape[0]
    d = _empty((nq, r), np.float64, q)
    i = _empty((nq, r), np.int64, q)
    c = _empty((nq,), np.int32, q)
    dev.ctx.check(_fn(dev.ctx, "pqs_derived_search", f64)(dev.ctx.handle, dev.handle, full.handle, dd.handle, ptr(q),
                                                            nq, int(r), int(r2), ptr(d), ptr(i), ptr(c),
                                                            _io(dev.ctx, q, d)), "derived_search")
    return d, i, c


def search_two_pass(dpq: DerivedPQ, db: CodeList, query: np.ndarray, r: int, r2: int) -> NeighborSet:
    """derived.py:402-409: quantized derived-table candidate scan, then the
    exact rerank of the admitted candidates; the r best by (distance, id)."""
    query = np.asarray(query)
    if query.ndim != 1 or query.shape[0] != dpq.pq.d:
        raise ValueError(f"query must have shape ({dpq.pq.d},)")
    d, i, c = search_two_pass_batch(dpq, db, query[None, :], r, r2)
    n = int(c[0])
    return NeighborSet.from_pairs(r, d[0, :n], i[0, :n])


# ------------------------------------------------------------ files (derived.py:412-449)
def write_derived_body(f: BinaryIO, dpq: DerivedPQ) -> None:
    write_quantizer_body(f, dpq.pq)
    _write_i32(f, dpq.bbar)
    _write_array(f, dpq.derived, "<f4")


def read_derived_body(f: BinaryIO) -> DerivedPQ:
    pq = read_quantizer_body(f)
    bbar = _read_i32(f)
    derived = _read_array(f, "<f4", pq.m * (1 << bbar) * pq.dsub)
    return DerivedPQ(pq=pq, bbar=bbar, derived=derived.reshape(pq.m, 1 << bbar, pq.dsub))


def save_derived(path, dpq: DerivedPQ) -> None:
    with open(path, "wb") as f:
        write_derived_body(f, dpq)


def load_derived(path) -> DerivedPQ:
    with open(path, "rb") as f:
        return read_derived_body(f)


def load_quantizer_any(path):
    """derived.py:437-449: a DerivedPQ when the derived extension follows."""
    with open(path, "rb") as f:
        pq = read_quantizer_body(f)
        peek = f.read(4)
        if len(peek) < 4:
            return pq
        (bbar,) = struct.unpack("<i", peek)
        derived = _read_array(f, "<f4", pq.m * (1 << bbar) * pq.dsub)
        return DerivedPQ(pq=pq, bbar=bbar, derived=derived.reshape(pq.m, 1 << bbar, pq.dsub))
