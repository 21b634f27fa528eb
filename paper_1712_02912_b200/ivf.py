"""Drop-in for `pqscan.ivf.query_ivf` (ivf.py:148-196), kernels 'adc' and
'quick-adc', on the GPU.

Probes (nearest_k, _dist.py:42-67) and the list scans run in libpqs.so
(K7 probe GEMM + exact fp64 re-score, K8 list-major filtered scan, K6 exact
residual-table rerank, K5 select; kernel='quick-adc': the per-list Quick ADC of ivf_qadc.cu;
kernel='derived': the per-list two-pass search of derived.cu).  The index is
uploaded once and cached on the IvfIndex object.
"""

from __future__ import annotations

import numpy as np

from ._cache import device_cached, freeze
from .engine import DeviceIvf
from .types import IvfIndex, NeighborSet

KERNELS = ("adc", "quick-adc", "derived")   # ivf.py:46
DEFAULT_R2_SMALL = 9000                     # ivf.py:47
DEFAULT_R2_LARGE = 120000                   # ivf.py:48


def default_r2(r: int) -> int:
    """ivf.py:51-53."""
    return DEFAULT_R2_SMALL if r <= 100 else DEFAULT_R2_LARGE


def device_index(index: IvfIndex) -> DeviceIvf:
    """The index's device copy: rebuilt after any rebinding of a sealed
    container's field or change to index.lists (mutation epoch); every list's
    codes/ids are frozen when uploaded (in-place edits raise)."""
    def build():
        for lst in index.lists:
            freeze(lst.codes)
            freeze(lst.ids)
        return DeviceIvf(index)

    return device_cached(index, "_pqs_ivf", (index.coarse, index.pq.codebooks, id(index.lists), len(index.lists)),
                         build)


def query_ivf(index: IvfIndex, query: np.ndarray, ma: int, r: int, kernel: str = "adc",
              init_count: int = 200, r2: int | None = None) -> NeighborSet:
    """ivf.py:148-196, kernels 'adc', 'quick-adc' and 'derived'."""
    kernel = kernel.replace("_", "-")
    if kernel not in KERNELS:
        raise ValueError(f"kernel must be one of {KERNELS}")
    if not 1 <= ma <= index.K:
        raise ValueError(f"ma must be in [1, {index.K}]")
    if r < 1:
        raise ValueError("r must be >= 1")
    if kernel == "quick-adc" and (index.pq.b != 4 or index.pq.m % 2):
        raise ValueError("quick-adc kernel requires b=4 and even m")
    if kernel == "derived" and index.dpq is None:
        raise ValueError("index has no derived quantizer")
    query = np.asarray(query, dtype=np.float64)
    if query.shape != (index.d,):
        raise ValueError(f"query must have shape ({index.d},)")
    dev = device_index(index)
    if kernel == "quick-adc" and init_count < 1:
        # qadc_scan raises at the first non-empty probed list (quickadc.py:123-124)
        cells, _ = dev.probe(query[None, :], int(ma))
        if any(index.lists[int(c)].n for c in cells[0]):
            raise ValueError("init_count must be >= 1")
        return NeighborSet(r)

    d, i, c = dev.search(query[None, :], int(ma), int(r), kernel=kernel,
                         init_count=int(init_count), r2=(r2 if r2 is not None else default_r2(r)), dpq=index.dpq)
    n = int(c[0])
    return NeighborSet.from_pairs(r, d[0, :n], i[0, :n])


def query_ivf_batch(index: IvfIndex, queries: np.ndarray, ma: int, r: int, kernel: str = "adc",
                    init_count: int = 200):
    """Batched query_ivf: (nq, d) -> (dist (nq, r), ids (nq, r), count (nq,))."""
    kernel = kernel.replace("_", "-")
    if kernel == "derived" and index.dpq is None:
        raise ValueError("index has no derived quantizer")
    return device_index(index).search(queries, int(ma), int(r), kernel=kernel, init_count=int(init_count),
                                      r2=default_r2(r), dpq=index.dpq)
