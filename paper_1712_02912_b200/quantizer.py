"""Drop-in for `pqscan.quantizer.encode` (quantizer.py:308-325) on the GPU.

Per sub-space the index of the nearest centroid by the fp64 direct-difference
distance summed in scipy's order (nearest, _dist.py:24-39), ties to the lowest
index -- computed by encode_kernel (csrc/encode.cu), bit-identical.  Like the
reference (pq.rotate casts to float64) the kernel reads the rows in fp64:
float32 rows go through pqs_encode, every other dtype is cast to float64 and
goes through pqs_encode_f64 -- nothing is rounded to float32.
"""

from __future__ import annotations

import numpy as np

from .types import ProductQuantizer


def encode(pq: ProductQuantizer, x: np.ndarray) -> np.ndarray:
    """quantizer.py:308-325 -- (d,) -> (m,) or (n, d) -> (n, m) uint8 codes."""
    from .scan import _device_quantizer

    x = np.asarray(x)
    single = x.ndim == 1
    rows = x[None, :] if single else x
    if rows.shape[1] != pq.d:
        raise ValueError(f"vector dimensionality {rows.shape[1]}, expected {pq.d}")
    if pq.b > 8:
        raise NotImplementedError("device encode supports b <= 8 (uint8 codes)")
    out = _device_quantizer(pq).encode(rows)
    return out[0] if single else out
