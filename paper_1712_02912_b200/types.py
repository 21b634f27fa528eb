"""Host-side containers with the reference's names, fields and validation.

Mirrors `pqscan` (arxiv/paper_1712_02912): ProductQuantizer
(quantizer.py:38-89), LookupTables / NeighborSet / CodeList /
TransposedCodeList (scan.py:21-245), QuantParams (fastscan.py:28-45),
QuantizedTables4 (quickadc.py:32-54), IvfIndex (ivf.py:58-86).  These are
plain data holders; all compute on them runs on the GPU (paper_1712_02912_b200.scan,
.quickadc, .ivf).
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field

import numpy as np

BINS = 127                     # fastscan.py:23
BLOCK = 16                     # scan.py:206
DEFAULT_INIT_COUNT = 200       # quickadc.py:28
DEFAULT_INIT_COUNT_BILLION = 1000  # quickadc.py:29


# ---------------------------------------------------------------------------
# device-cache coherence.  The drop-in functions upload a container's arrays
# to the GPU once and reuse the device copy (paper_1712_02912_b200/_cache.py).
# The reference recomputes from the arrays on every call, so two things would
# otherwise make results stale: (1) in-place edits of a cached array -- the
# cache makes every array it uploads read-only, so such edits raise
# (numpy's "assignment destination is read-only"): refused, loudly; (2)
# rebinding a field (`codelist.codes = other`, `index.lists[c] = other`) --
# sealed containers bump a global mutation epoch that every cache key holds.
_EPOCH = [0]


def mutation_epoch() -> int:
    """Bumped whenever a field of a sealed container is rebound."""
    return _EPOCH[0]


class _Sealable:
    def __setattr__(self, name, value):
        if self.__dict__.get("_sealed", False) and not name.startswith("_"):
            _EPOCH[0] += 1
        object.__setattr__(self, name, value)

    def _seal(self):
        object.__setattr__(self, "_sealed", True)


class _TrackedList(list):
    """IvfIndex.lists: a list whose mutations bump the mutation epoch."""

    def _bump(self):
        _EPOCH[0] += 1


for _name in ("__setitem__", "__delitem__", "__iadd__", "__imul__", "append", "extend", "insert", "pop",
              "remove", "clear", "sort", "reverse"):
    def _make(fn):
        def wrapped(self, *a, **k):
            self._bump()
            return fn(self, *a, **k)
        wrapped.__name__ = fn.__name__
        return wrapped
    setattr(_TrackedList, _name, _make(getattr(list, _name)))


class TrainError(RuntimeError):
    """quantizer.py:21-22."""


@dataclass
class ProductQuantizer(_Sealable):
    """quantizer.py:38-89: m codebooks of 2^b centroids over d/m dims."""

    m: int
    b: int
    d: int
    codebooks: np.ndarray
    rotation: np.ndarray | None = None

    def __post_init__(self):
        if self.d % self.m != 0:
            raise ValueError(f"d={self.d} not divisible by m={self.m}")
        if not 1 <= self.b <= 16:
            raise ValueError(f"b={self.b} out of range [1, 16]")
        k, dsub = 1 << self.b, self.d // self.m
        self.codebooks = np.ascontiguousarray(self.codebooks, dtype=np.float32)
        if self.codebooks.shape != (self.m, k, dsub):
            raise ValueError(f"codebooks shape {self.codebooks.shape}, expected {(self.m, k, dsub)}")
        if not np.all(np.isfinite(self.codebooks)):
            raise ValueError("codebooks contain non-finite values")
        if self.rotation is not None:
            self.rotation = np.ascontiguousarray(self.rotation, dtype=np.float32)
            if self.rotation.shape != (self.d, self.d):
                raise ValueError("rotation must be d x d")
        self._seal()

    @property
    def k(self) -> int:
        return 1 << self.b

    @property
    def dsub(self) -> int:
        return self.d // self.m

    @property
    def code_dtype(self) -> np.dtype:
        return np.dtype(np.uint8 if self.b <= 8 else np.uint16)


@dataclass
class LookupTables:
    """scan.py:21-42: per-sub-space squared distances, (m, 2^b) float32."""

    tables: np.ndarray

    def __post_init__(self):
        self.tables = np.ascontiguousarray(self.tables, dtype=np.float32)
        if self.tables.ndim != 2:
            raise ValueError("tables must be 2-D (m, 2^b)")

    @property
    def m(self) -> int:
        return self.tables.shape[0]

    @property
    def k(self) -> int:
        return self.tables.shape[1]

    @property
    def nbytes(self) -> int:
        return self.tables.nbytes


def implicit_ids(obj) -> bool:
    """True while obj.ids is still the arange the container made itself
    (CodeList default ids, scan.py:170-171): the device then uses id = index."""
    imp = obj.__dict__.get("_implicit_ids")
    return imp is not None and imp is obj.ids


class NeighborSet:
    """scan.py:84-139: the r smallest (distance, id) pairs; lower id on ties."""

    __slots__ = ("r", "_heap")

    def __init__(self, r: int):
        if r < 1:
            raise ValueError("r must be >= 1")
        self.r = r
        self._heap: list[tuple[float, int]] = []

    def __len__(self) -> int:
        return len(self._heap)

    @property
    def worst(self) -> float:
        if len(self._heap) < self.r:
            return float("inf")
        return -self._heap[0][0]

    def push(self, distance: float, ident: int) -> bool:
        entry = (-float(distance), -int(ident))
        if len(self._heap) < self.r:
            heapq.heappush(self._heap, entry)
            return True
        if entry > self._heap[0]:
            heapq.heappushpop(self._heap, entry)
            return True
        return False

    def items(self) -> list[tuple[float, int]]:
        return sorted((-d, -i) for d, i in self._heap)

    def to_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        pairs = self.items()
        return (np.array([p[0] for p in pairs], dtype=np.float64),
                np.array([p[1] for p in pairs], dtype=np.int64))

    @classmethod
    def from_pairs(cls, r: int, dists, ids) -> "NeighborSet":
        out = cls(r)
        out._heap = [(-float(d), -int(i)) for d, i in zip(dists[:r], ids[:r])]
        heapq.heapify(out._heap)
        return out


@dataclass
class CodeList(_Sealable):
    """scan.py:157-194: codes (n, m) uint8/uint16 with parallel int64 ids."""

    codes: np.ndarray
    ids: np.ndarray | None = None

    def __post_init__(self):
        self.codes = np.ascontiguousarray(self.codes)
        if self.codes.ndim != 2:
            raise ValueError("codes must be 2-D (n, m)")
        if self.codes.dtype not in (np.dtype(np.uint8), np.dtype(np.uint16)):
            raise ValueError("codes must be uint8 or uint16")
        implicit = self.ids is None
        if self.ids is None:
            self.ids = np.arange(self.codes.shape[0], dtype=np.int64)
        else:
            self.ids = np.ascontiguousarray(self.ids, dtype=np.int64)
        if self.ids.shape != (self.codes.shape[0],):
            raise ValueError("ids length must match codes")
        # the default arange ids are implicit on the device (id = index) for as
        # long as this very array is the list's ids (see implicit_ids)
        self._implicit_ids = self.ids if implicit else None
        self._seal()

    @property
    def n(self) -> int:
        return self.codes.shape[0]

    @property
    def m(self) -> int:
        return self.codes.shape[1]


@dataclass
class TransposedCodeList(_Sealable):
    """scan.py:209-245: codes regrouped into component-major blocks of 16."""

    blocks: np.ndarray
    n: int
    m: int
    b: int
    ids: np.ndarray

    def __post_init__(self):
        self.blocks = np.ascontiguousarray(self.blocks, dtype=np.uint8)
        self.ids = np.ascontiguousarray(self.ids, dtype=np.int64)
        rows = self.m // 2 if self.b == 4 else self.m
        nblocks = (self.n + BLOCK - 1) // BLOCK
        if self.blocks.shape != (nblocks, rows, BLOCK):
            raise ValueError(f"blocks shape {self.blocks.shape}, expected {(nblocks, rows, BLOCK)}")
        if self.ids.shape != (self.n,):
            raise ValueError("ids length must match n")
        self._implicit_ids = None
        self._seal()

    @property
    def n_blocks(self) -> int:
        return self.blocks.shape[0]

    def block_validity(self, block_index: int) -> int:
        if block_index < self.n_blocks - 1:
            return BLOCK
        return self.n - block_index * BLOCK


@dataclass
class QuantParams:
    """fastscan.py:28-45: 127-bin range; values >= qmax map to 127."""

    qmin: float
    qmax: float

    def __post_init__(self):
        if not (math.isfinite(self.qmin) and math.isfinite(self.qmax)):
            raise ValueError("quantization bounds must be finite")
        if self.qmax < self.qmin:
            raise ValueError("qmax must be >= qmin")

    @property
    def scale(self) -> float:
        span = self.qmax - self.qmin
        return BINS / span if span > 0.0 else 0.0


@dataclass
class QuantizedTables4:
    """quickadc.py:32-54: m 16-entry uint8 tables in [0, 127] + range."""

    tables: np.ndarray
    params: QuantParams

    def __post_init__(self):
        self.tables = np.ascontiguousarray(self.tables, dtype=np.uint8)
        if self.tables.ndim != 2 or self.tables.shape[1] != 16:
            raise ValueError("quantized tables must have shape (m, 16)")
        if np.any(self.tables > BINS):
            raise ValueError("quantized entries must be <= 127")

    @property
    def m(self) -> int:
        return self.tables.shape[0]

    def rescale(self, bins) -> np.ndarray | float:
        p = self.params
        v = np.asarray(bins, dtype=np.float64) * (p.qmax - p.qmin) / BINS + p.qmin
        return float(v[()]) if v.ndim == 0 else v


@dataclass
class IvfIndex(_Sealable):
    """ivf.py:58-86: coarse centroids, residual quantizer, K inverted lists."""

    coarse: np.ndarray
    pq: ProductQuantizer
    lists: list
    dpq: object | None = None
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        self.coarse = np.ascontiguousarray(self.coarse, dtype=np.float32)
        if self.coarse.ndim != 2 or self.coarse.shape[1] != self.pq.d:
            raise ValueError("coarse centroids must have shape (K, d)")
        if len(self.lists) != self.coarse.shape[0]:
            raise ValueError("need exactly one inverted list per coarse centroid")
        if self.dpq is not None and self.dpq.pq is not self.pq:
            raise ValueError("derived quantizer must wrap the index quantizer")
        self.lists = self.lists  # as a _TrackedList
        self._seal()

    def __setattr__(self, name, value):
        if name == "lists" and not isinstance(value, _TrackedList):
            value = _TrackedList(value)
        super().__setattr__(name, value)

    @property
    def K(self) -> int:
        return self.coarse.shape[0]

    @property
    def d(self) -> int:
        return self.coarse.shape[1]

    @property
    def n(self) -> int:
        return sum(lst.n for lst in self.lists)
