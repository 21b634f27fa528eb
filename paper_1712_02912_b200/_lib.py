"""ctypes binding of libpqs.so (include/pqs.h).

The library is the product: every search in this package runs through it on
the GPU.  There is no CPU fallback -- if the library or a CUDA device is
missing, calls raise `RuntimeError` (loudly, by design).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PQS_LIB", os.path.join(_HERE, "lib", "libpqs.so"))

PQS_OK = 0
PQS_ERR_INVALID = 1
PQS_ERR_CUDA = 2
PQS_ERR_NOMEM = 3
PQS_ERR_UNSUPPORTED = 4
IO_HOST = 0
IO_DEVICE = 1

OPT_CAND_CAP = 1
OPT_SAMPLE_DIV = 2
OPT_FORCE_FALLBACK = 3
OPT_SCAN4_ENGINE = 4
OPT_TC_CHUNK_TILES = 5
OPT_SCAN8_ENGINE = 6
OPT_IVF_ENGINE = 7
STAT_LAUNCHES = 1
STAT_LAST_MAX_CAND = 2
STAT_LAST_OVERFLOW = 3
STAT_LAST_EVALS = 4
STAT_LAST_SCAN_NS = 5
STAT_LAST_SCAN_LAUNCHES = 6
STAT_LAST_CAND_TOTAL = 7
STAT_LAST_SCAN_ENGINE = 8
STAT_LAST_SCAN_WORK = 9
STAT_LAST_RERANK_TOTAL = 10
STAT_LAST_SLOT_EVALS = 11

_p = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_d = ctypes.c_double

# name -> (restype, argtypes); mirrors include/pqs.h exactly
SIGNATURES = {
    "pqs_api_version": (_i, []),
    "pqs_ctx_create": (_i, [_i, ctypes.POINTER(_p)]),
    "pqs_ctx_destroy": (None, [_p]),
    "pqs_ctx_set_stream": (_i, [_p, _p]),
    "pqs_ctx_synchronize": (_i, [_p]),
    "pqs_ctx_set_option": (_i, [_p, _i, _i64]),
    "pqs_ctx_get_stat": (_i, [_p, _i, ctypes.POINTER(_i64)]),
    "pqs_last_error": (ctypes.c_char_p, [_p]),
    "pqs_pq_create": (_i, [_p, _i, _i, _i, _p, ctypes.POINTER(_p)]),
    "pqs_pq_destroy": (None, [_p]),
    "pqs_db_create": (_i, [_p, _p, _i64, _i, _i, _p, _i64, _i, ctypes.POINTER(_p)]),
    "pqs_db_set_prefix": (_i, [_p, _p, _p, _i64, _i]),
    "pqs_db_create_packed": (_i, [_p, _p, _i64, _i, _i, _i, _p, _i64, _i, ctypes.POINTER(_p)]),
    "pqs_db_destroy": (None, [_p]),
    "pqs_compute_tables": (_i, [_p, _p, _p, _i64, _p, _i]),
    "pqs_scan_distances": (_i, [_p, _p, _p, _i64, _i, _p, _i]),
    "pqs_adc_scan": (_i, [_p, _p, _p, _i64, _i, _i, _p, _p, _p, _i]),
    "pqs_adc_search": (_i, [_p, _p, _p, _p, _i64, _i, _p, _p, _p, _i]),
    "pqs_qadc_scan": (_i, [_p, _p, _p, _i64, _i, _i, _p, _p, _p, _p, _p, _i]),
    "pqs_qadc_search": (_i, [_p, _p, _p, _p, _i64, _i, _i, _p, _p, _p, _p, _p, _i]),
    "pqs_quantized_distances": (_i, [_p, _p, _p, _i64, _p, _i]),
    "pqs_quantize": (_i, [_p, _d, _d, _p, _i64, _p, _i]),
    "pqs_ivf_create": (_i, [_p, _p, _p, _i64, _p, _p, _p, _i, ctypes.POINTER(_p)]),
    "pqs_encode": (_i, [_p, _p, _p, _i64, _p, _i64, _p, _p, _i]),
    "pqs_ivf_destroy": (None, [_p]),
    "pqs_ivf_probe": (_i, [_p, _p, _p, _i64, _i, _p, _p, _i]),
    "pqs_ivf_search": (_i, [_p, _p, _p, _i64, _i, _i, _p, _p, _p, _i]),
    "pqs_ivf_qadc_search": (_i, [_p, _p, _p, _i64, _i, _i, _i, _p, _p, _p, _i]),
    "pqs_fastscan_checked": (_i, [_p, _p, _p, _i64, _i64, _i, _p, _i]),
    "pqs_derived_search": (_i, [_p, _p, _p, _p, _p, _i64, _i, _i64, _p, _p, _p, _i]),
    "pqs_ivf_derived_search": (_i, [_p, _p, _p, _p, _i64, _i, _i, _i64, _p, _p, _p, _i]),
    "pqs_nearest": (_i, [_p, _p, _i64, _i, _p, _i64, _p, _p, _i]),
    "pqs_merge_topr": (_i, [_p, _i, _p, _p, _p, _i64, _i, _i, _p, _p, _p, _i]),
}
# float64 twins of the query-taking entry points (same arguments; queries double*)
F64_TWINS = ("pqs_compute_tables", "pqs_adc_search", "pqs_qadc_search", "pqs_ivf_probe", "pqs_ivf_search",
             "pqs_ivf_qadc_search", "pqs_derived_search", "pqs_ivf_derived_search", "pqs_encode", "pqs_nearest")
for _n in F64_TWINS:
    SIGNATURES[_n + "_f64"] = SIGNATURES[_n]

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | None = None):
    """Load libpqs.so and declare every exported symbol.  Raises if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(
                f"libpqs.so not found at {p}: build it with `make` (or __graft_entry__.build()); "
                "this package has no CPU fallback"
            )
        lib = ctypes.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


class PQSError(RuntimeError):
    pass


def ptr(a) -> int | None:
    """Address of a numpy array or a torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


class Context:
    """One CUDA device + stream of the engine (pqs_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = ctypes.c_void_p()
        st = self.lib.pqs_ctx_create(int(device), ctypes.byref(h))
        if st != PQS_OK:
            raise PQSError(f"pqs_ctx_create(device={device}) failed with status {st} (no CUDA device?)")
        self.handle = h
        self.device = int(device)
        self.follow_torch = True   # device-array calls run on torch's current stream
        self._bound = None

    def check(self, status: int, what: str = "") -> None:
        if status == PQS_OK:
            return
        msg = self.lib.pqs_last_error(self.handle).decode(errors="replace")
        if status == PQS_ERR_INVALID:
            raise ValueError(msg)
        if status == PQS_ERR_UNSUPPORTED:
            raise NotImplementedError(f"{what}: {msg}")
        raise PQSError(f"{what}: {msg} (status {status})")

    def set_stream(self, stream_ptr: int | None) -> None:
        """Issue this context's work on a CUDA stream: a cudaStream_t handle
        (torch.cuda.Stream.cuda_stream; 0 = the legacy default stream), or
        None for the context's own stream.  Disables following torch."""
        self.follow_torch = False
        self._set(stream_ptr)

    def _set(self, stream_ptr):
        # 0 is torch's (legacy) default stream: pass cudaStreamLegacy, since a
        # NULL handle selects the context's own stream in the C ABI
        handle = None if stream_ptr is None else (1 if int(stream_ptr) == 0 else int(stream_ptr))
        self.check(self.lib.pqs_ctx_set_stream(self.handle, handle), "set_stream")
        self._bound = stream_ptr

    def bind_torch_stream(self) -> None:
        """Before a call on CUDA tensors: run on torch's current stream of this
        device, so the call is ordered with the kernels that produced its
        inputs and those that consume its outputs."""
        if not self.follow_torch:
            return
        import torch

        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != self._bound:
            self._set(s)

    def synchronize(self) -> None:
        self.check(self.lib.pqs_ctx_synchronize(self.handle), "synchronize")

    def set_option(self, option: int, value: int) -> None:
        self.check(self.lib.pqs_ctx_set_option(self.handle, option, int(value)), "set_option")

    def stat(self, which: int) -> int:
        out = ctypes.c_int64()
        self.check(self.lib.pqs_ctx_get_stat(self.handle, which, ctypes.byref(out)), "get_stat")
        return int(out.value)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.pqs_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_default = {}
_default_lock = threading.Lock()


def default_context(device: int | None = None) -> Context:
    """Process-wide context per device (device 0 unless PQS_DEVICE is set)."""
    if device is None:
        device = int(os.environ.get("PQS_DEVICE", "0"))
    with _default_lock:
        ctx = _default.get(device)
        if ctx is None:
            ctx = Context(device)
            _default[device] = ctx
        return ctx
