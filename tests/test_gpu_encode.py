"""GPU: encode (quantizer.py:308-325) bit-exact against the reference's golden
codes (plain and IVF residual, incl. tied centroids), and device-built code
lists / indexes (io = device) equal the host-built ones."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O
from tests.helpers import encode, kmeans_books, mixture

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _pq(books):
    m, k, dsub = books.shape
    return P.ProductQuantizer(m, int(np.log2(k)), m * dsub, books)


@pytest.mark.parametrize("tag", ["c1", "c3", "c2"])
def test_encode_golden(golden, tag):
    g = golden("encode.npz")
    pq = _pq(g[f"{tag}_codebooks"])
    np.testing.assert_array_equal(P.encode(pq, g[f"{tag}_x"]), g[f"{tag}_codes"])
    np.testing.assert_array_equal(P.encode(pq, g[f"{tag}_x"][3]), g[f"{tag}_codes"][3])
    dq = P.DeviceQuantizer(pq)
    got = dq.encode(g[f"{tag}_x"], coarse=g[f"{tag}_coarse"], cells=g[f"{tag}_cells"])
    np.testing.assert_array_equal(got, g[f"{tag}_rescodes"])


def test_encode_device_tensors_and_oracle():
    import torch

    rng = np.random.default_rng(5)
    x = mixture(rng, 40_000, 96, comps=64, hi=1.0, sigma=0.3)
    books = kmeans_books(x[:5000], 16, 16, iters=3)
    pq = _pq(books)
    want = O.encode(books, x[:3000])
    np.testing.assert_array_equal(P.encode(pq, x[:3000]), want)
    dq = P.DeviceQuantizer(pq)
    xt = torch.from_numpy(x).cuda()
    got = dq.encode(xt)
    assert got.is_cuda
    np.testing.assert_array_equal(got[:3000].cpu().numpy(), want)
    with pytest.raises(ValueError):
        P.encode(pq, x[:, :95])
    # float64 rows are encoded from their float64 values (quantizer.py:319-323)
    x64 = x[:500].astype(np.float64) + 1e-4 * np.random.default_rng(9).normal(size=(500, 96))
    np.testing.assert_array_equal(P.encode(pq, x64), O.encode(books, x64))


def test_device_built_codes_equal_host_built():
    import torch

    rng = np.random.default_rng(6)
    x = mixture(rng, 200_000, 64, comps=64)
    books = kmeans_books(x[:10000], 16, 16, iters=3)
    pq = _pq(books)
    qs = mixture(np.random.default_rng(7), 64, 64, comps=64)
    dq = P.DeviceQuantizer(pq)
    codes_dev = dq.encode(torch.from_numpy(x).cuda())
    codes_host = codes_dev.cpu().numpy()
    a = P.DeviceCodes(codes_host, 4).qadc_search(dq, qs, 200, 50)
    b = P.DeviceCodes(codes_dev, 4).qadc_search(dq, qs, 200, 50)
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)
    # b = 8 layout from device codes (tile transpose kernel)
    books8 = kmeans_books(x[:10000], 8, 256, iters=2)
    pq8 = _pq(books8)
    dq8 = P.DeviceQuantizer(pq8)
    c8 = dq8.encode(torch.from_numpy(x[:50_000]).cuda())
    a = P.DeviceCodes(c8.cpu().numpy(), 8).adc_search(dq8, qs, 30)
    b = P.DeviceCodes(c8, 8).adc_search(dq8, qs, 30)
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)
    with pytest.raises(ValueError):
        P.DeviceCodes(torch.full((100, 16), 16, dtype=torch.uint8, device="cuda"), 4)


def test_ivf_from_device_arrays(golden):
    import torch

    g = golden("ivf.npz")
    m, k, dsub = g["codebooks"].shape
    pq = P.ProductQuantizer(m, int(np.log2(k)), m * dsub, g["codebooks"])
    host = P.DeviceIvf.from_arrays(pq, g["coarse"], g["list_sizes"], g["list_codes"], g["list_ids"])
    dev = P.DeviceIvf.from_arrays(pq, torch.from_numpy(g["coarse"]).cuda(), g["list_sizes"],
                                  torch.from_numpy(g["list_codes"]).cuda(), torch.from_numpy(g["list_ids"]).cuda())
    for ma, r in [(4, 50), (16, 100)]:
        a = host.search(g["queries"], ma, r)
        b = dev.search(g["queries"], ma, r)
        for u, v in zip(a, b):
            np.testing.assert_array_equal(u, v)
        d, i, c = a
        for qi in range(g["queries"].shape[0]):
            n = int(c[qi])
            np.testing.assert_array_equal(d[qi, :n], g[f"ma{ma}_r{r}_dist"][qi][:n])
            np.testing.assert_array_equal(i[qi, :n], g[f"ma{ma}_r{r}_ids"][qi][:n])
