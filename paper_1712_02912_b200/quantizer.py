"""Drop-in for `pqscan.quantizer.encode` (quantizer.py:308-325) on the GPU.

Per sub-space the index of the nearest centroid by the fp64 direct-difference
distance summed in scipy's order (nearest, _dist.py:24-39), ties to the lowest
index -- computed by encode_kernel (csrc/encode.cu), bit-identical.  The
device path takes float32 vectors: float64 input is accepted when it is
exactly representable in float32 (the reference's own data is float32), and
rejected otherwise rather than silently rounded.
"""

from __future__ import annotations

import numpy as np

from .types import ProductQuantizer


def as_f32_exact(x, what: str) -> np.ndarray:
    """float32 view of x; float64 values must round-trip exactly."""
    x = np.asarray(x)
    if x.dtype == np.float32:
        return np.ascontiguousarray(x)
    x32 = x.astype(np.float32)
    if not np.array_equal(x32.astype(x.dtype), x, equal_nan=True):
        raise NotImplementedError(f"{what}: the device path computes from float32 inputs; "
                                  f"these values are not exactly representable in float32")
    return np.ascontiguousarray(x32)


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
    out = _device_quantizer(pq).encode(as_f32_exact(rows, "encode"))
    return out[0] if single else out
