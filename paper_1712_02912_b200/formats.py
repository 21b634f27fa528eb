"""Persistence formats of the reference -> host objects and device handles
(SURVEY 8f row 2).

Byte-compatible readers/writers of the reference's little-endian formats:
PQZ1 quantizers (quantizer.py:345-381), PQL1 code lists (scan.py:290-359,
nibble packing for b <= 4 at scan.py:293-316) and IVF1 indexes
(ivf.py:199-229), with the reference's error behaviour (`FormatError`, a
ValueError carrying the byte offset, _binio.py:11-18).  The device loaders
parse only the headers on the host and hand the code payload to
`pqs_db_create_packed`, which uploads the packed bytes as they are in the file
(b <= 4: half the bytes) and unpacks them on the GPU into the scan layouts.
IVF1 files with a derived quantizer (has_derived) carry a DerivedPQ.
"""

from __future__ import annotations

import ctypes
import struct
from typing import BinaryIO

import numpy as np

from ._lib import IO_HOST, default_context, ptr
from .types import CodeList, IvfIndex, ProductQuantizer

MAGIC_QUANTIZER = b"PQZ1"
MAGIC_CODES = b"PQL1"
MAGIC_IVF = b"IVF1"


class FormatError(ValueError):
    """_binio.py:11-18 -- malformed file content, with the byte offset."""

    def __init__(self, message: str, offset: int | None = None):
        if offset is not None:
            message = f"{message} (byte offset {offset})"
        super().__init__(message)
        self.offset = offset


# ------------------------------------------------------------ primitives
def _expect_magic(f: BinaryIO, magic: bytes) -> None:
    off = f.tell()
    got = f.read(4)
    if got != magic:
        raise FormatError(f"bad magic {got!r}, expected {magic!r}", offset=off)


def _read(f: BinaryIO, fmt: str, what: str):
    size = struct.calcsize(fmt)
    off = f.tell()
    raw = f.read(size)
    if len(raw) != size:
        raise FormatError(f"truncated {what} field", offset=off)
    return struct.unpack(fmt, raw)[0]


def _read_i32(f: BinaryIO) -> int:
    return _read(f, "<i", "int32")


def _read_array(f: BinaryIO, dtype: str, count: int) -> np.ndarray:
    dt = np.dtype(dtype)
    off = f.tell()
    raw = f.read(dt.itemsize * count)
    if len(raw) != dt.itemsize * count:
        raise FormatError(f"truncated array, wanted {count} items of {dt}", offset=off)
    return np.frombuffer(raw, dtype=dt).copy()


def _write_i32(f: BinaryIO, v: int) -> None:
    f.write(struct.pack("<i", int(v)))


def _write_array(f: BinaryIO, arr, dtype: str) -> None:
    f.write(np.ascontiguousarray(arr, dtype=np.dtype(dtype)).tobytes())


# ------------------------------------------------------------ PQZ1
def write_quantizer_body(f: BinaryIO, pq: ProductQuantizer) -> None:
    f.write(MAGIC_QUANTIZER)
    for v in (pq.m, pq.b, pq.d, 1 if pq.rotation is not None else 0):
        _write_i32(f, v)
    if pq.rotation is not None:
        _write_array(f, pq.rotation, "<f4")
    _write_array(f, pq.codebooks, "<f4")


def read_quantizer_body(f: BinaryIO) -> ProductQuantizer:
    _expect_magic(f, MAGIC_QUANTIZER)
    m, b, d, has_rot = _read_i32(f), _read_i32(f), _read_i32(f), _read_i32(f)
    rotation = _read_array(f, "<f4", d * d).reshape(d, d) if has_rot else None
    k, dsub = 1 << b, d // m
    books = _read_array(f, "<f4", m * k * dsub).reshape(m, k, dsub)
    return ProductQuantizer(m=m, b=b, d=d, codebooks=books, rotation=rotation)


def save_quantizer(path, pq: ProductQuantizer) -> None:
    with open(path, "wb") as f:
        write_quantizer_body(f, pq)


def load_quantizer(path) -> ProductQuantizer:
    with open(path, "rb") as f:
        return read_quantizer_body(f)


# ------------------------------------------------------------ PQL1
def _payload_spec(n: int, m: int, b: int) -> tuple[int, str]:
    if b <= 4:
        return n * ((m + 1) // 2), "u1"
    if b <= 8:
        return n * m, "u1"
    return n * m, "<u2"


def pack_codes(codes: np.ndarray, b: int) -> np.ndarray:
    """scan.py:293-305: b <= 4 -> even component in the low nibble."""
    n, m = codes.shape
    if b <= 4:
        out = np.zeros((n, (m + 1) // 2), dtype=np.uint8)
        out |= codes[:, 0::2].astype(np.uint8)
        odd = codes[:, 1::2].astype(np.uint8)
        out[:, :odd.shape[1]] |= odd << 4
        return out
    return codes.astype(np.uint8 if b <= 8 else np.uint16)


def unpack_codes(raw: np.ndarray, n: int, m: int, b: int) -> np.ndarray:
    """scan.py:308-316."""
    if b <= 4:
        packed = raw.reshape(n, (m + 1) // 2)
        codes = np.empty((n, m), dtype=np.uint8)
        codes[:, 0::2] = packed & 0x0F
        codes[:, 1::2] = (packed >> 4)[:, :m // 2]
        return codes
    return raw.reshape(n, m).astype(np.uint8 if b <= 8 else np.uint16)


def write_codes_body(f: BinaryIO, codelist: CodeList, b: int) -> None:
    n, m = codelist.n, codelist.m
    if np.any(codelist.codes.astype(np.int64) >= (1 << b)):
        raise ValueError(f"codes exceed b={b}")
    f.write(MAGIC_CODES)
    for v in (n, m, b, 1):
        _write_i32(f, v)
    _write_array(f, pack_codes(codelist.codes, b), "<u2" if b > 8 else "u1")
    _write_array(f, codelist.ids, "<i8")


def _read_codes_header(f: BinaryIO) -> tuple[int, int, int, int]:
    _expect_magic(f, MAGIC_CODES)
    return _read_i32(f), _read_i32(f), _read_i32(f), _read_i32(f)


def read_codes_body(f: BinaryIO) -> tuple[CodeList, int]:
    n, m, b, has_ids = _read_codes_header(f)
    count, dtype = _payload_spec(n, m, b)
    codes = unpack_codes(_read_array(f, dtype, count), n, m, b)
    ids = _read_array(f, "<i8", n) if has_ids else None
    return CodeList(codes, ids), b


def save_codes(path, codelist: CodeList, b: int) -> None:
    with open(path, "wb") as f:
        write_codes_body(f, codelist, b)


def load_codes(path) -> tuple[CodeList, int]:
    with open(path, "rb") as f:
        return read_codes_body(f)


# ------------------------------------------------------------ IVF1
def save_ivf(path, index: IvfIndex) -> None:
    with open(path, "wb") as f:
        f.write(MAGIC_IVF)
        _write_i32(f, index.K)
        _write_i32(f, 1 if index.dpq is not None else 0)
        if index.dpq is not None:
            from .derived import write_derived_body

            write_derived_body(f, index.dpq)
        else:
            write_quantizer_body(f, index.pq)
        _write_array(f, index.coarse, "<f4")
        for lst in index.lists:
            write_codes_body(f, lst, index.pq.b)


def _read_ivf_head(f: BinaryIO):
    _expect_magic(f, MAGIC_IVF)
    K = _read_i32(f)
    dpq = None
    if _read_i32(f):
        from .derived import read_derived_body

        dpq = read_derived_body(f)
        pq = dpq.pq
    else:
        pq = read_quantizer_body(f)
    coarse = _read_array(f, "<f4", K * pq.d).reshape(K, pq.d)
    return K, pq, coarse, dpq


def load_ivf(path) -> IvfIndex:
    with open(path, "rb") as f:
        K, pq, coarse, dpq = _read_ivf_head(f)
        lists = [read_codes_body(f)[0] for _ in range(K)]
    return IvfIndex(coarse=coarse, pq=pq, lists=lists, dpq=dpq)


# ------------------------------------------------------------ device handles
def load_codes_device(path, layout_b: int | None = None, id_base: int = 0, ctx=None):
    """PQL1 file -> (DeviceCodes, b): the payload is uploaded as stored and
    unpacked on the GPU (pqs_db_create_packed).  layout_b: 4 (Quick ADC) or 8
    (float ADC); default 4 for b <= 4 with even m, else 8.  Ids stored in the
    file are kept; a file written with implicit ids (0..n-1) keeps implicit
    ids on the device."""
    from .engine import DeviceCodes

    ctx = ctx or default_context()
    with open(path, "rb") as f:
        n, m, b, has_ids = _read_codes_header(f)
        if b > 8:
            raise NotImplementedError("device code lists hold b <= 8 components")
        count, dtype = _payload_spec(n, m, b)
        payload = _read_array(f, dtype, count)
        ids = _read_array(f, "<i8", n) if has_ids else None
    if layout_b is None:
        layout_b = 4 if (b <= 4 and m % 2 == 0 and m <= 32) else 8
    if ids is not None and np.array_equal(ids, np.arange(n, dtype=np.int64)):
        ids = None  # implicit ids: the strict Quick ADC threshold applies
    elif ids is not None:
        ids = np.ascontiguousarray(ids)
    h = ctypes.c_void_p()
    ctx.check(ctx.lib.pqs_db_create_packed(ctx.handle, ptr(payload), n, m, b, layout_b, ptr(ids), int(id_base),
                                           IO_HOST, ctypes.byref(h)), "db_create_packed")
    db = DeviceCodes.__new__(DeviceCodes)
    db.ctx, db.handle, db.n, db.m, db.b = ctx, h, n, m, layout_b
    return db, b


def load_ivf_device(path, ctx=None):
    """IVF1 file -> DeviceIvf (lists concatenated in cell order on the host)."""
    from .engine import DeviceIvf

    with open(path, "rb") as f:
        K, pq, coarse, _dpq = _read_ivf_head(f)
        sizes = np.empty(K, dtype=np.int64)
        codes, ids = [], []
        for c in range(K):
            cl, _ = read_codes_body(f)
            sizes[c] = cl.n
            codes.append(cl.codes)
            ids.append(cl.ids)
    allc = np.ascontiguousarray(np.concatenate(codes) if K else np.zeros((0, pq.m), np.uint8), dtype=np.uint8)
    alli = np.ascontiguousarray(np.concatenate(ids) if K else np.zeros(0, np.int64), dtype=np.int64)
    return DeviceIvf.from_arrays(pq, coarse, sizes, allc, alli, ctx=ctx)


__all__ = ["FormatError", "save_quantizer", "load_quantizer", "save_codes", "load_codes", "save_ivf", "load_ivf",
           "load_codes_device", "load_ivf_device", "pack_codes", "unpack_codes"]
