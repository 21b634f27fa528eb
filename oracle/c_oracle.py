"""ctypes binding of oracle/lib/libpqs_oracle.so (oracle/qadc_oracle.c) --
TEST INFRASTRUCTURE ONLY (tests/ use it for oracle checks at BASELINE size).

pack_nibbles: PQL1 4-bit packing (scan.py:293-316).  qadc_topr: the r
smallest (bin, id) of quantized_distances (quickadc.py:87-101) +
_select_best (scan.py:142-154) for ids = id_base + position."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "lib", "libpqs_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", _LIB, os.path.join(_HERE, "qadc_oracle.c")],
                           check=True)
        L = ctypes.CDLL(_LIB)
        p, i64, i = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.pqo_qdist_packed.argtypes = [p, i64, i, p, p]
        L.pqo_qdist_packed.restype = None
        L.pqo_qadc_topr_packed.argtypes = [p, i64, i, p, i64, i, p, p, p]
        L.pqo_qadc_topr_packed.restype = i64
        L.pqo_merge_topr.argtypes = [i, p, p, p, i64, i, p, p]
        L.pqo_merge_topr.restype = i64
        _lib = L
    return _lib


def pack_nibbles(codes: np.ndarray) -> np.ndarray:
    """(n, m) components < 16, m even -> (n, m/2): 2j low nibble, 2j+1 high (scan.py:293-316)."""
    c = np.asarray(codes, dtype=np.uint8)
    return np.ascontiguousarray(c[:, 0::2] | (c[:, 1::2] << 4))


def qdist(packed: np.ndarray, m: int, qtables: np.ndarray) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    qt = np.ascontiguousarray(qtables, dtype=np.uint8)
    out = np.empty(packed.shape[0], np.uint8)
    lib().pqo_qdist_packed(packed.ctypes.data, packed.shape[0], m, qt.ctypes.data, out.ctypes.data)
    return out


def qadc_topr(packed: np.ndarray, m: int, qtables: np.ndarray, r: int, id_base: int = 0, scratch: bool = False):
    """-> (bins uint8 ascending, ids int64) of the r smallest (bin, id)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    qt = np.ascontiguousarray(qtables, dtype=np.uint8)
    n = packed.shape[0]
    ob = np.empty(min(r, n), np.uint8)
    oi = np.empty(min(r, n), np.int64)
    sc = np.empty(n, np.uint8) if scratch else None
    k = lib().pqo_qadc_topr_packed(packed.ctypes.data, n, m, qt.ctypes.data, int(id_base), int(r),
                                   None if sc is None else sc.ctypes.data, ob.ctypes.data, oi.ctypes.data)
    return ob[:k], oi[:k]


def merge_topr(bins_list, ids_list, r: int):
    G = len(bins_list)
    stride = max(len(b) for b in bins_list)
    B = np.zeros((G, stride), np.uint8)
    I = np.zeros((G, stride), np.int64)
    C = np.array([len(b) for b in bins_list], np.int64)
    for g in range(G):
        B[g, :C[g]] = bins_list[g]
        I[g, :C[g]] = ids_list[g]
    ob = np.empty(r, np.uint8)
    oi = np.empty(r, np.int64)
    k = lib().pqo_merge_topr(G, B.ctypes.data, I.ctypes.data, C.ctypes.data, stride, r, ob.ctypes.data,
                             oi.ctypes.data)
    return ob[:k], oi[:k]
