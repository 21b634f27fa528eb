"""CPU-only: libpqs.so loads and exports exactly the C ABI declared in include/pqs.h."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pqs.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pqs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_api():
    fns = header_functions()
    assert "pqs_adc_scan" in fns and "pqs_qadc_scan" in fns and "pqs_ivf_search" in fns
    assert len(fns) >= 25


def test_library_exports_every_symbol():
    from paper_1712_02912_b200 import _lib

    lib = _lib.load_library()
    for name in header_functions():
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_python_binding_covers_header():
    from paper_1712_02912_b200 import _lib

    assert set(header_functions()) == set(_lib.SIGNATURES)


def test_api_version():
    from paper_1712_02912_b200 import _lib

    assert _lib.load_library().pqs_api_version() == 3


def test_f64_twins():
    """Every query-taking entry point has a float64 twin (the reference
    computes from float64(query), quantizer.py:85-89)."""
    fns = set(header_functions())
    from paper_1712_02912_b200 import _lib

    for name in _lib.F64_TWINS:
        assert name in fns and name + "_f64" in fns, name


def test_no_library_gemm_linked():
    """The probe GEMM is hand-written tcgen05 (probe.cu): libpqs.so links no cuBLAS."""
    import subprocess

    from paper_1712_02912_b200 import _lib

    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "cublas" not in out


def test_no_device_fails_loudly():
    """Without a GPU the product path raises; it never falls back to the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1712_02912_b200 import _lib

    with pytest.raises(_lib.PQSError):
        _lib.Context(0)


def test_reference_names_exported():
    import paper_1712_02912_b200 as P

    for name in ["compute_tables", "scan", "scan_distances", "adc_distance", "transpose_blocks",
                 "detranspose_blocks", "qadc_scan", "qadc_block", "quantize", "quantize_tables_4bit",
                 "quantized_distances", "query_ivf", "CodeList", "NeighborSet", "LookupTables",
                 "IvfIndex", "ProductQuantizer", "QuantParams", "QuantizedTables4", "TransposedCodeList",
                 "BINS", "BLOCK", "DEFAULT_INIT_COUNT", "KERNELS", "default_r2"]:
        assert hasattr(P, name), name
