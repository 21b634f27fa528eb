"""CPU-only: pin the C restatement of the Quick ADC steps (oracle/qadc_oracle.c,
used for oracle checks at BASELINE size) to the real reference's golden
outputs and to the numpy oracle."""

import numpy as np

from oracle import c_oracle as C
from oracle import pqscan_oracle as O


def test_c_oracle_golden(golden):
    g = golden("quick_adc.npz")
    codes, books, qs = g["codes"], g["codebooks"], g["queries"]
    packed = C.pack_nibbles(codes)
    for s in range(6):
        init, r = int(g[f"s{s}_init"]), int(g[f"s{s}_r"])
        for qi, q in enumerate(qs):
            t = O.compute_tables(books, q)
            qmin, qmax = O.qadc_params(t, codes, init, r)
            qt = O.quantize(qmin, qmax, t)
            np.testing.assert_array_equal(qt, g[f"s{s}_qtables"][qi])
            for scratch in (False, True):
                b, i = C.qadc_topr(packed, codes.shape[1], qt, r, scratch=scratch)
                n = len(b)
                np.testing.assert_array_equal(b, g[f"s{s}_bins"][qi][:n])
                np.testing.assert_array_equal(i, g[f"s{s}_ids"][qi][:n])


def test_c_oracle_vs_numpy_ties_saturation_and_merge():
    rng = np.random.default_rng(8)
    for n, m, r, hi in [(5000, 16, 100, 3), (3000, 8, 4000, 16), (20000, 16, 250, 2), (777, 4, 50, 16)]:
        codes = rng.integers(0, hi, (n, m)).astype(np.uint8)
        qt = rng.integers(0, 128, (m, 16)).astype(np.uint8)
        if n == 3000:
            qt[:] = 120                      # heavy saturation at 127
        ref = O.quantized_distances(codes, qt)
        np.testing.assert_array_equal(C.qdist(C.pack_nibbles(codes), m, qt), ref)
        ob, oi = O.select_best(ref.astype(np.float64), np.arange(n, dtype=np.int64) + 1000, r)
        b, i = C.qadc_topr(C.pack_nibbles(codes), m, qt, r, id_base=1000)
        np.testing.assert_array_equal(b, ob.astype(np.uint8))
        np.testing.assert_array_equal(i, oi)
        # shards merged == unsharded (global ids)
        parts = [(lo, min(n, lo + 999)) for lo in range(0, n, 999)]
        res = [C.qadc_topr(C.pack_nibbles(codes[lo:hi_]), m, qt, r, id_base=1000 + lo) for lo, hi_ in parts]
        mb, mi = C.merge_topr([x[0] for x in res], [x[1] for x in res], r)
        np.testing.assert_array_equal(mb, b)
        np.testing.assert_array_equal(mi, i)
