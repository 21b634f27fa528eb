"""GPU: fast_scan (fastscan.py:328-386) through libpqs.so -- neighbour sets
and ScanStats identical to the reference (golden) and to the oracle's
sequential pruned scan at a larger size; build_small_tables/lower_bound
consistent with the device's lower bounds."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from paper_1712_02912_b200 import fastscan as F
from tests.helpers import encode, kmeans_books, mixture
from tests.test_fastscan_host import SETTINGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _grouped(g):
    return F.GroupedDatabase(g["g_keys"], g["g_offsets"], g["g_counts"], g["g_packed"], g["g_ids"])


@pytest.mark.parametrize("init,r", SETTINGS)
def test_fast_scan_golden(golden, init, r):
    g = golden("fastscan.npz")
    gr = _grouped(g)
    pq = P.ProductQuantizer(8, 8, 32, g["codebooks"])
    tag = f"i{init}_r{r}"
    for qi, q in enumerate(g["queries"]):
        nset, st = P.fast_scan(gr, P.compute_tables(pq, q), init, r)
        items = nset.items()
        n = len(items)
        assert [d for d, _ in items] == g[f"{tag}_dist"][qi][:n].tolist()
        assert [i for _, i in items] == g[f"{tag}_ids"][qi][:n].tolist()
        assert (st.total, st.checked, st.pruned) == tuple(g[f"{tag}_stats"][qi])


def test_fast_scan_errors(golden):
    g = golden("fastscan.npz")
    gr = _grouped(g)
    t = P.compute_tables(P.ProductQuantizer(8, 8, 32, g["codebooks"]), g["queries"][0])
    for init in (0.0, 1.5):
        with pytest.raises(ValueError):
            P.fast_scan(gr, t, init, 10)
    with pytest.raises(ValueError):
        P.fast_scan(gr, t, 0.1, 0)


def test_fast_scan_vs_oracle_large():
    """200k codes, 12 queries, batched statistics vs the sequential oracle."""
    rng = np.random.default_rng(5)
    x = mixture(rng, 200_000, 64, comps=64)
    books = kmeans_books(x[:20000], 8, 256, iters=3)
    codes = encode(books, x)
    ids = rng.permutation(10**6)[:200_000].astype(np.int64)
    gr = F.group_codes(P.CodeList(codes, ids))
    sc, si = gr.reconstruct_codes(), gr.ids
    pq = P.ProductQuantizer(8, 8, 64, books)
    qs = x[rng.choice(200_000, 12, replace=False)] + rng.normal(0, 3, (12, 64)).astype(np.float32)
    tabs = P.compute_tables_batch(pq, qs)
    for init, r in [(0.01, 100), (0.002, 1000)]:
        checked = F.fast_scan_checked(gr._device(), tabs, int(np.ceil(init * 200_000)), r)
        for qi in (0, 5, 11):
            od, oi, oc, op = O.fast_scan(sc, si, tabs[qi], init, r)
            nset, st = P.fast_scan(gr, P.LookupTables(tabs[qi]), init, r)
            assert [d for d, _ in nset.items()] == od.tolist()
            assert [i for _, i in nset.items()] == oi.tolist()
            assert st.checked == oc == int(checked[qi]) and st.pruned == op


def test_small_tables_bound(golden):
    g = golden("fastscan.npz")
    pq = P.ProductQuantizer(8, 8, 32, g["codebooks"])
    t = P.compute_tables(pq, g["queries"][1])
    params = P.compute_quant_params(t, P.CodeList(g["codes"], g["ids"]), 0.01, 100)
    qmin, qmax = O.qadc_params(t.tables, g["codes"], 200, 100)
    assert params.qmin == qmin
    for c in g["codes"][:40]:
        small = P.build_small_tables(t, params, P.group_key(c))
        lb = P.lower_bound(small, P.pack_code(c))
        qd = O.quantize(params.qmin, params.qmax, np.array([O.adc_distance(t.tables, c)]))[0]
        assert lb <= qd
