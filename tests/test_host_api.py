"""CPU-only host logic: container validation and error behaviour mirror the reference."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P


def test_neighborset_semantics():
    ns = P.NeighborSet(2)
    for ident in (9, 4, 7):
        ns.push(1.5, ident)
    assert ns.items() == [(1.5, 4), (1.5, 7)]
    assert ns.worst == 1.5
    with pytest.raises(ValueError):
        P.NeighborSet(0)


def test_codelist_validation():
    with pytest.raises(ValueError):
        P.CodeList(np.zeros((3,), np.uint8))
    with pytest.raises(ValueError):
        P.CodeList(np.zeros((3, 2), np.int32))
    with pytest.raises(ValueError):
        P.CodeList(np.zeros((3, 2), np.uint8), np.arange(2))
    cl = P.CodeList(np.zeros((3, 2), np.uint8))
    np.testing.assert_array_equal(cl.ids, np.arange(3))


def test_quant_params_validation():
    with pytest.raises(ValueError):
        P.QuantParams(1.0, 0.0)
    with pytest.raises(ValueError):
        P.QuantParams(float("nan"), 1.0)
    assert P.QuantParams(0.0, 0.0).scale == 0.0
    assert P.QuantParams(0.0, 127.0).scale == 1.0


def test_rescale():
    qt = P.QuantizedTables4(np.zeros((2, 16), np.uint8), P.QuantParams(10.0, 137.0))
    assert qt.rescale(0) == pytest.approx(10.0)
    assert qt.rescale(127) == pytest.approx(137.0)


def test_transpose_round_trip_and_layout(golden):
    g = golden("quick_adc.npz")
    cl = P.CodeList(g["codes"])
    t = P.transpose_blocks(cl, 4)
    np.testing.assert_array_equal(t.blocks, g["blocks"])
    back = P.detranspose_blocks(t)
    np.testing.assert_array_equal(back.codes, g["codes"])
    # test_scan.py:155-163 known answer
    codes = np.array([[1, 2, 3, 4], [5, 6, 7, 8]], dtype=np.uint8)
    tl = P.transpose_blocks(P.CodeList(codes), 4)
    assert tl.blocks[0, 0, 0] == (2 << 4) | 1 and tl.blocks[0, 1, 1] == (8 << 4) | 7
    with pytest.raises(ValueError):
        P.transpose_blocks(P.CodeList(np.zeros((2, 3), np.uint8)), 4)


def test_query_validation_before_device():
    pq = P.ProductQuantizer(2, 4, 4, np.zeros((2, 16, 2), np.float32))
    idx = P.IvfIndex(np.zeros((3, 4), np.float32), pq, [P.CodeList(np.zeros((0, 2), np.uint8))] * 3)
    with pytest.raises(ValueError):
        P.query_ivf(idx, np.zeros(4), ma=1, r=1, kernel="nope")
    with pytest.raises(ValueError):
        P.query_ivf(idx, np.zeros(4), ma=4, r=1)
    with pytest.raises(ValueError):
        P.query_ivf(idx, np.zeros(4), ma=1, r=1, kernel="derived")
    assert P.default_r2(100) == 9000 and P.default_r2(101) == 120000
