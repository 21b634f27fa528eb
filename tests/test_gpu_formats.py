"""GPU: device handles loaded straight from reference-written files (PQL1
payload uploaded as stored and unpacked on the device; IVF1) search exactly
like handles built from the decoded arrays."""

import os

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _path(name):
    return os.path.join(GOLDEN, name)


def _same(a, b):
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)


def test_packed_quick_adc_list(golden):
    g = golden("formats.npz")
    pq = P.load_quantizer(_path("fmt_pq4.pqz"))
    dq = P.DeviceQuantizer(pq)
    db, b = P.load_codes_device(_path("fmt_codes4.pql"))
    assert b == 4 and db.b == 4
    qs = np.random.default_rng(2).normal(64, 30, (20, 32)).astype(np.float32)
    _same(db.qadc_search(dq, qs, 50, 30), P.DeviceCodes(g["codes4"], 4).qadc_search(dq, qs, 50, 30))


def test_float_lists_with_ids_and_odd_m(golden):
    g = golden("formats.npz")
    pq = P.load_quantizer(_path("fmt_pq8.pqz"))
    dq = P.DeviceQuantizer(pq)
    qs = np.random.default_rng(3).normal(64, 30, (20, 32)).astype(np.float32)
    db, b = P.load_codes_device(_path("fmt_codes8.pql"))
    assert b == 8 and db.b == 8
    _same(db.adc_search(dq, qs, 40), P.DeviceCodes(g["codes8"], 8, ids=g["ids8"]).adc_search(dq, qs, 40))
    # b = 3, m = 5: nibble-packed payload, odd m -> float layout
    books3 = np.random.default_rng(4).normal(0, 1, (5, 8, 2)).astype(np.float32)
    pq3 = P.ProductQuantizer(5, 3, 10, books3)
    db3, b3 = P.load_codes_device(_path("fmt_codes3.pql"))
    assert b3 == 3 and db3.b == 8
    t = P.DeviceQuantizer(pq3).compute_tables(np.random.default_rng(5).normal(0, 1, (7, 10)).astype(np.float32))
    _same(db3.adc_scan(t, 12), P.DeviceCodes(g["codes3"], 8).adc_scan(t, 12))


def test_ivf_file(golden):
    g = golden("formats.npz")
    ivf = P.load_ivf_device(_path("fmt_index.ivf"))
    ref = P.DeviceIvf(P.load_ivf(_path("fmt_index.ivf")))
    qs = np.random.default_rng(6).normal(64, 30, (9, 32)).astype(np.float32)
    _same(ivf.search(qs, 4, 25), ref.search(qs, 4, 25))
