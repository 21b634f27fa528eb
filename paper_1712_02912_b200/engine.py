"""Device handles and the batched search API over libpqs.so.

The reference (`pqscan`) searches one query per call; the GPU needs batches.
These classes own device copies of a quantizer / code list / inverted index
and search many queries per call.  Arrays may be numpy (host; copies happen
inside the call) or CUDA torch tensors (device; zero-copy, same stream rules
as the context).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import IO_DEVICE, IO_HOST, default_context, ptr


def _is_device(x) -> bool:
    return not isinstance(x, np.ndarray) and getattr(x, "is_cuda", False)


def _io_of(*arrays) -> int:
    dev = [_is_device(a) for a in arrays if a is not None]
    if dev and all(dev):
        return IO_DEVICE
    if any(dev):
        raise ValueError("mix of host and device arrays in one call")
    return IO_HOST


def _io(ctx, *arrays) -> int:
    """io flag of a call; device calls are bound to torch's current stream."""
    io = _io_of(*arrays)
    if io == IO_DEVICE:
        ctx.bind_torch_stream()
    return io


def _empty(shape, dtype, like):
    if _is_device(like):
        import torch

        tmap = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32,
                np.uint8: torch.uint8, np.float32: torch.float32}
        return torch.empty(shape, dtype=tmap[dtype], device=like.device)
    return np.empty(shape, dtype=dtype)


def _check_out(out, shapes, dtypes, like):
    """Validate caller-provided output arrays (same side as `like`, C-contiguous)."""
    if len(out) != len(shapes):
        raise ValueError("out must hold one array per result")
    for o, shp, dt in zip(out, shapes, dtypes):
        if _is_device(o) != _is_device(like):
            raise ValueError("out arrays must live on the same side (host / device) as the queries")
        if tuple(o.shape) != tuple(shp):
            raise ValueError(f"out array of shape {tuple(o.shape)}, expected {tuple(shp)}")
        if _is_device(o):
            if not o.is_contiguous() or str(o.dtype) != "torch." + np.dtype(dt).name:
                raise ValueError("out tensors must be contiguous with the result dtypes")
        elif o.dtype != np.dtype(dt) or not o.flags["C_CONTIGUOUS"]:
            raise ValueError("out arrays must be C-contiguous with the result dtypes")
    return out


def _queries(a, ndim, what):
    """Query / vector rows and whether they are float64.  float32 rows stay
    float32; every other dtype becomes float64 -- the reference computes from
    float64(query) (quantizer.py:85-89, ivf.py:170, quantizer.py:319-323), and
    the *_f64 entry points read it as given (nothing is rounded to float32)."""
    if _is_device(a):
        if str(a.dtype) not in ("torch.float32", "torch.float64") or not a.is_contiguous():
            raise ValueError(f"{what} must be a contiguous float32 or float64 tensor")
        if a.dim() != ndim:
            raise ValueError(f"{what} must be {ndim}-D")
        return a, str(a.dtype) == "torch.float64"
    a = np.asarray(a)
    if a.dtype != np.float32:
        a = a.astype(np.float64)
    a = np.ascontiguousarray(a)
    if a.ndim != ndim:
        raise ValueError(f"{what} must be {ndim}-D")
    return a, a.dtype == np.float64


def _fn(ctx, name, f64):
    return getattr(ctx.lib, name + "_f64" if f64 else name)


def _host_f32(a, ndim, what):
    """Lookup tables (LookupTables forces float32, scan.py:21-42) and other
    float32-by-definition inputs."""
    if _is_device(a):
        if a.dtype.__str__() != "torch.float32" or not a.is_contiguous():
            raise ValueError(f"{what} must be a contiguous float32 tensor")
        if a.dim() != ndim:
            raise ValueError(f"{what} must be {ndim}-D")
        return a
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim != ndim:
        raise ValueError(f"{what} must be {ndim}-D")
    return a


def nearest(points, centroids, ctx=None):
    """nearest (_dist.py:24-39), the assignment step of build_ivf (ivf.py:122):
    per point (index of its nearest centroid, squared distance to it) by the
    fp64 cdist sum, ties to the lowest index -- pqs_nearest: the tcgen05 tf32
    probe GEMM's certified shortlist, re-scored exactly in fp64.  points (n, d)
    float32 / float64, host array or CUDA tensor; centroids (K, d) float32 on
    the same side.  Returns (idx int64 (n,), dist float64 (n,))."""
    ctx = ctx or default_context()
    x, f64 = _queries(points, 2, "points")
    if _is_device(x):
        if not _is_device(centroids) or str(centroids.dtype) != "torch.float32" or centroids.dim() != 2:
            raise ValueError("centroids must be a 2-D float32 CUDA tensor when the points are on the device")
        c = centroids.contiguous()
    else:
        c = np.ascontiguousarray(centroids, dtype=np.float32)
        if c.ndim != 2:
            raise ValueError("centroids must be 2-D")
    if tuple(c.shape)[1] != x.shape[1]:
        raise ValueError("points and centroids must have the same dimension")
    n = x.shape[0]
    idx = _empty((n,), np.int64, x)
    dist = _empty((n,), np.float64, x)
    ctx.check(_fn(ctx, "pqs_nearest", f64)(ctx.handle, ptr(c), c.shape[0], c.shape[1], ptr(x), n, ptr(idx),
                                            ptr(dist), _io(ctx, x, idx)), "nearest")
    return idx, dist


class DeviceQuantizer:
    """pqs_pq: device copy of a ProductQuantizer's codebooks (no rotation)."""

    def __init__(self, pq, ctx=None):
        if pq.rotation is not None:
            raise NotImplementedError("rotated (OPQ) quantizers are outside the device scan path")
        if pq.b > 8:
            raise NotImplementedError("device tables support b <= 8")
        self.ctx = ctx or default_context()
        self.m, self.b, self.d, self.k = pq.m, pq.b, pq.d, pq.k
        books = np.ascontiguousarray(pq.codebooks, dtype=np.float32)
        h = ctypes.c_void_p()
        self.ctx.check(self.ctx.lib.pqs_pq_create(self.ctx.handle, pq.m, pq.b, pq.d, ptr(books), ctypes.byref(h)),
                       "pq_create")
        self.handle = h

    def compute_tables(self, queries):
        """Batched compute_tables (scan.py:45-56): (nq, d) -> (nq, m, k) fp32."""
        q, f64 = _queries(queries, 2, "queries")
        if q.shape[1] != self.d:
            raise ValueError(f"queries must have shape (nq, {self.d})")
        out = _empty((q.shape[0], self.m, self.k), np.float32, q)
        self.ctx.check(_fn(self.ctx, "pqs_compute_tables", f64)(self.ctx.handle, self.handle, ptr(q), q.shape[0],
                                                                  ptr(out), _io(self.ctx, q, out)), "compute_tables")
        return out

    def encode(self, x, coarse=None, cells=None):
        """encode (quantizer.py:308-325) of (n, d) fp32 vectors -> (n, m) uint8,
        bit-identical; with coarse (K, d) and cells (n,) the IVF residuals
        x - coarse[cells] are encoded (build_ivf, ivf.py:137-140)."""
        x, f64 = _queries(x, 2, "vectors")
        if x.shape[1] != self.d:
            raise ValueError(f"vector dimensionality {x.shape[1]}, expected {self.d}")
        K = 0
        if coarse is not None:
            coarse = _host_f32(coarse, 2, "coarse")
            K = coarse.shape[0]
            if _is_device(cells):
                if str(cells.dtype) != "torch.int64" or cells.dim() != 1:
                    raise ValueError("device cells must be a 1-D int64 tensor")
                cells = cells.contiguous()
            else:
                cells = np.ascontiguousarray(cells, dtype=np.int64)
            if tuple(cells.shape) != (x.shape[0],):
                raise ValueError(f"cells must have shape ({x.shape[0]},)")
        out = _empty((x.shape[0], self.m), np.uint8, x)
        self.ctx.check(_fn(self.ctx, "pqs_encode", f64)(self.ctx.handle, self.handle, ptr(x), x.shape[0], ptr(coarse),
                                                          K, ptr(cells), ptr(out), _io(self.ctx, x, coarse, cells, out)),
                       "encode")
        return out

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.ctx.lib.pqs_pq_destroy(self.handle)
        except Exception:
            pass


class DeviceCodes:
    """pqs_db: a device-resident code list (b=8 float ADC or b=4 Quick ADC)."""

    def __init__(self, codes, b: int, ids=None, id_base: int = 0, ctx=None):
        """codes: (n, m) numpy array or contiguous CUDA uint8 tensor (built on the
        device, e.g. by DeviceQuantizer.encode); ids likewise (int64) or None."""
        self.ctx = ctx or default_context()
        if _is_device(codes):
            if str(codes.dtype) != "torch.uint8" or codes.dim() != 2 or not codes.is_contiguous():
                raise ValueError("device codes must be a contiguous 2-D uint8 tensor")
            if ids is not None and (not _is_device(ids) or str(ids.dtype) != "torch.int64" or not ids.is_contiguous()):
                raise ValueError("ids of device codes must be a contiguous int64 CUDA tensor")
            io = IO_DEVICE
            ids_arr = ids
            self.ctx.bind_torch_stream()
        else:
            codes = np.asarray(codes)
            if codes.ndim != 2:
                raise ValueError("codes must be 2-D (n, m)")
            if codes.size and int(codes.max()) > 255:
                raise NotImplementedError("device code lists hold components < 256")
            codes = np.ascontiguousarray(codes, dtype=np.uint8)
            ids_arr = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
            io = IO_HOST
        self.n, self.m, self.b = int(codes.shape[0]), int(codes.shape[1]), b
        h = ctypes.c_void_p()
        self.ctx.check(self.ctx.lib.pqs_db_create(self.ctx.handle, ptr(codes), self.n, self.m, b, ptr(ids_arr),
                                                  int(id_base), io, ctypes.byref(h)), "db_create")
        self.handle = h

    def set_prefix(self, prefix_codes):
        """Global Quick ADC prefix for a shard (quickadc.py:130-137)."""
        if _is_device(prefix_codes):
            p, io = prefix_codes.contiguous(), IO_DEVICE
            self.ctx.bind_torch_stream()
        else:
            p, io = np.ascontiguousarray(prefix_codes, dtype=np.uint8), IO_HOST
        self.ctx.check(self.ctx.lib.pqs_db_set_prefix(self.ctx.handle, self.handle, ptr(p), int(p.shape[0]), io),
                       "set_prefix")

    # -- float ADC (b=8) --------------------------------------------------
    def scan_distances(self, tables):
        t = _host_f32(tables, 3, "tables")
        out = _empty((t.shape[0], self.n), np.float64, t)
        self.ctx.check(self.ctx.lib.pqs_scan_distances(self.ctx.handle, self.handle, ptr(t), t.shape[0], t.shape[2],
                                                       ptr(out), _io(self.ctx, t, out)), "scan_distances")
        return out

    def adc_scan(self, tables, r: int):
        """scan() for a batch of tables (nq, m, k) -> (dist, ids, count)."""
        t = _host_f32(tables, 3, "tables")
        if t.shape[1] != self.m:
            raise ValueError(f"codes must have shape (n, {t.shape[1]})")
        nq = t.shape[0]
        d = _empty((nq, r), np.float64, t)
        i = _empty((nq, r), np.int64, t)
        c = _empty((nq,), np.int32, t)
        self.ctx.check(self.ctx.lib.pqs_adc_scan(self.ctx.handle, self.handle, ptr(t), nq, t.shape[2], int(r), ptr(d),
                                                 ptr(i), ptr(c), _io(self.ctx, t, d)), "adc_scan")
        return d, i, c

    def adc_search(self, dq: DeviceQuantizer, queries, r: int, out=None):
        """Batched compute_tables + scan: (nq, d) queries -> (dist, ids, count);
        out: optional caller-owned output arrays as in qadc_search."""
        q, f64 = _queries(queries, 2, "queries")
        nq = q.shape[0]
        if out is not None:
            d, i, c = _check_out(out, ((nq, r), (nq, r), (nq,)), (np.float64, np.int64, np.int32), q)
        else:
            d = _empty((nq, r), np.float64, q)
            i = _empty((nq, r), np.int64, q)
            c = _empty((nq,), np.int32, q)
        self.ctx.check(_fn(self.ctx, "pqs_adc_search", f64)(self.ctx.handle, self.handle, dq.handle, ptr(q), nq, int(r),
                                                              ptr(d), ptr(i), ptr(c), _io(self.ctx, q, d)), "adc_search")
        return d, i, c

    # -- Quick ADC (b=4) ---------------------------------------------------
    def qadc_scan(self, tables, init_count: int, r: int):
        """qadc_scan for a batch of tables (nq, m, 16) ->
        (bins uint8, ids, count, qtables (nq,m,16) uint8, qminmax (nq,2))."""
        t = _host_f32(tables, 3, "tables")
        if t.shape[2] != 16 or t.shape[1] != self.m:
            raise ValueError("tables do not match the code list shape")
        nq = t.shape[0]
        bins = _empty((nq, r), np.uint8, t)
        i = _empty((nq, r), np.int64, t)
        c = _empty((nq,), np.int32, t)
        qt = _empty((nq, self.m, 16), np.uint8, t)
        qmm = _empty((nq, 2), np.float64, t)
        self.ctx.check(self.ctx.lib.pqs_qadc_scan(self.ctx.handle, self.handle, ptr(t), nq, int(init_count), int(r),
                                                  ptr(bins), ptr(i), ptr(c), ptr(qt), ptr(qmm), _io(self.ctx, t, bins)),
                       "qadc_scan")
        return bins, i, c, qt, qmm

    def qadc_search(self, dq: DeviceQuantizer, queries, init_count: int, r: int, want_tables: bool = False,
                    out=None):
        """Batched compute_tables + qadc_scan.  out: optional caller-owned
        (bins uint8 (nq, r), ids int64 (nq, r), count int32 (nq,)) arrays on
        the queries' side (e.g. pinned host buffers reused across calls)."""
        q, f64 = _queries(queries, 2, "queries")
        nq = q.shape[0]
        if out is not None:
            bins, i, c = _check_out(out, ((nq, r), (nq, r), (nq,)), (np.uint8, np.int64, np.int32), q)
        else:
            bins = _empty((nq, r), np.uint8, q)
            i = _empty((nq, r), np.int64, q)
            c = _empty((nq,), np.int32, q)
        qt = _empty((nq, self.m, 16), np.uint8, q) if want_tables else None
        qmm = _empty((nq, 2), np.float64, q) if want_tables else None
        self.ctx.check(_fn(self.ctx, "pqs_qadc_search", f64)(self.ctx.handle, self.handle, dq.handle, ptr(q), nq,
                                                               int(init_count), int(r), ptr(bins), ptr(i), ptr(c),
                                                               ptr(qt), ptr(qmm), _io(self.ctx, q, bins)), "qadc_search")
        return bins, i, c, qt, qmm

    def quantized_distances(self, qtables):
        qt = qtables if _is_device(qtables) else np.ascontiguousarray(qtables, dtype=np.uint8)
        if qt.ndim != 3 or qt.shape[1] != self.m or qt.shape[2] != 16:
            raise ValueError(f"codes must have shape (n, {qt.shape[1]})")
        out = _empty((qt.shape[0], self.n), np.uint8, qt)
        self.ctx.check(self.ctx.lib.pqs_quantized_distances(self.ctx.handle, self.handle, ptr(qt), qt.shape[0],
                                                            ptr(out), _io(self.ctx, qt, out)), "quantized_distances")
        return out

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.ctx.lib.pqs_db_destroy(self.handle)
        except Exception:
            pass


class DeviceIvf:
    """pqs_ivf: device-resident IVFADC index (coarse + residual PQ + lists)."""

    def __init__(self, index, ctx=None):
        sizes = np.array([lst.n for lst in index.lists], dtype=np.int64)
        m = index.pq.m
        if sizes.sum():
            codes = np.ascontiguousarray(np.concatenate([np.asarray(l.codes).reshape(-1, m) for l in index.lists]),
                                         dtype=np.uint8)
            ids = np.ascontiguousarray(np.concatenate([l.ids for l in index.lists]), dtype=np.int64)
        else:
            codes = np.zeros((0, m), np.uint8)
            ids = np.zeros(0, np.int64)
        self._create(index.pq, np.ascontiguousarray(index.coarse, dtype=np.float32), sizes, codes, ids, ctx)

    @classmethod
    def from_arrays(cls, pq, coarse, list_sizes, codes, ids, ctx=None):
        """Index from lists already concatenated in cell order: coarse (K, d)
        fp32, list_sizes (K,) int64 (host), codes (n, m) uint8, ids (n,) int64
        -- numpy arrays or CUDA tensors (e.g. an index built on the device)."""
        self = cls.__new__(cls)
        if not _is_device(coarse):
            coarse = np.ascontiguousarray(coarse, dtype=np.float32)
        self._create(pq, coarse, np.ascontiguousarray(list_sizes, dtype=np.int64), codes, ids, ctx)
        return self

    def _create(self, pq, coarse, sizes, codes, ids, ctx):
        self.ctx = ctx or default_context()
        self.dq = DeviceQuantizer(pq, self.ctx)
        self.K, self.d = int(coarse.shape[0]), int(coarse.shape[1])
        self.n = int(np.asarray(sizes).sum())
        if sizes.shape != (self.K,):
            raise ValueError("list_sizes must have one entry per coarse centroid")
        h = ctypes.c_void_p()
        self.ctx.check(self.ctx.lib.pqs_ivf_create(self.ctx.handle, self.dq.handle, ptr(coarse), self.K, ptr(sizes),
                                                   ptr(codes), ptr(ids), _io(self.ctx, coarse, codes, ids),
                                                   ctypes.byref(h)), "ivf_create")
        self.handle = h

    def probe(self, queries, ma: int):
        q, f64 = _queries(queries, 2, "queries")
        nq = q.shape[0]
        cells = _empty((nq, ma), np.int64, q)
        dist = _empty((nq, ma), np.float64, q)
        self.ctx.check(_fn(self.ctx, "pqs_ivf_probe", f64)(self.ctx.handle, self.handle, ptr(q), nq, int(ma),
                                                             ptr(cells), ptr(dist), _io(self.ctx, q, cells)),
                       "ivf_probe")
        return cells, dist

    def search(self, queries, ma: int, r: int, kernel: str = "adc", init_count: int = 200, r2: int = 9000,
               dpq=None, out=None):
        """Batched query_ivf: kernel 'adc' (exact fp64 distances), 'quick-adc'
        (per-list Quick ADC bins rescaled to fp64, ivf.py:185-190) or 'derived'
        (ivf.py:191-195).  out: optional caller-owned (dist, ids, count) arrays."""
        q, f64 = _queries(queries, 2, "queries")
        if q.shape[1] != self.d:
            raise ValueError(f"query must have shape ({self.d},)")
        nq = q.shape[0]
        if out is not None:
            d, i, c = _check_out(out, ((nq, r), (nq, r), (nq,)), (np.float64, np.int64, np.int32), q)
        else:
            d = _empty((nq, r), np.float64, q)
            i = _empty((nq, r), np.int64, q)
            c = _empty((nq,), np.int32, q)
        io = _io(self.ctx, q, d)
        if kernel == "adc":
            st = _fn(self.ctx, "pqs_ivf_search", f64)(self.ctx.handle, self.handle, ptr(q), nq, int(ma), int(r),
                                                        ptr(d), ptr(i), ptr(c), io)
        elif kernel == "quick-adc":
            st = _fn(self.ctx, "pqs_ivf_qadc_search", f64)(self.ctx.handle, self.handle, ptr(q), nq, int(ma),
                                                             int(r), int(init_count), ptr(d), ptr(i), ptr(c), io)
        elif kernel == "derived":
            if dpq is None:
                raise ValueError("index has no derived quantizer")
            _, dd = dpq._device()
            st = _fn(self.ctx, "pqs_ivf_derived_search", f64)(self.ctx.handle, self.handle, dd.handle, ptr(q), nq,
                                                                int(ma), int(r), int(r2), ptr(d), ptr(i), ptr(c), io)
        else:
            raise ValueError(f"unknown device IVF kernel {kernel!r}")
        self.ctx.check(st, "ivf_search")
        return d, i, c

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.ctx.lib.pqs_ivf_destroy(self.handle)
        except Exception:
            pass


def merge_topr(dists, ids, counts, r: int, ctx=None):
    """Top-r of G per-shard lists by (distance, id): dists/ids (G, nq, r_in),
    counts (G, nq) -> (dist (nq, r), ids, count)."""
    ctx = ctx or default_context()
    if _is_device(dists):
        G, nq, r_in = dists.shape
    else:
        dists = np.ascontiguousarray(dists, dtype=np.float64)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        G, nq, r_in = dists.shape
    od = _empty((nq, r), np.float64, dists)
    oi = _empty((nq, r), np.int64, dists)
    oc = _empty((nq,), np.int32, dists)
    ctx.check(ctx.lib.pqs_merge_topr(ctx.handle, G, ptr(dists), ptr(ids), ptr(counts), nq, r_in, int(r), ptr(od),
                                     ptr(oi), ptr(oc), _io(ctx, dists, od)), "merge_topr")
    return od, oi, oc


def quantize_device(qmin: float, qmax: float, values, ctx=None):
    """fastscan.quantize (fastscan.py:48-57) on the GPU, fp64."""
    ctx = ctx or default_context()
    v = np.ascontiguousarray(values, dtype=np.float64)
    flat = v.reshape(-1)
    out = np.empty(flat.shape, dtype=np.uint8)
    ctx.check(ctx.lib.pqs_quantize(ctx.handle, float(qmin), float(qmax), ptr(flat), flat.shape[0], ptr(out), IO_HOST),
              "quantize")
    return out.reshape(v.shape)


__all__ = ["DeviceQuantizer", "DeviceCodes", "DeviceIvf", "merge_topr", "quantize_device", "_lib"]
