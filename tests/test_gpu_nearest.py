"""pqs_nearest against nearest (_dist.py:24-39): index and fp64 distance of the
nearest centroid, ties to the lowest index; the assignment step of build_ivf
(ivf.py:122)."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from oracle import pqscan_oracle as O

pytestmark = pytest.mark.gpu


def _ref(points, centroids):
    idx, dist = O.nearest_k(np.asarray(points, np.float64), np.asarray(centroids, np.float32), 1)
    return idx[:, 0], dist[:, 0]


@pytest.mark.parametrize("n,K,d,dtype", [(5000, 1000, 32, np.float32), (3000, 4096, 128, np.float64),
                                         (257, 3, 8, np.float32), (1000, 300, 300, np.float32)])
def test_nearest_matches_reference(n, K, d, dtype):
    rng = np.random.default_rng(n + K)
    cent = rng.normal(0, 4, (K, d)).astype(np.float32)
    pts = (cent[rng.integers(0, K, n)] + rng.normal(0, 2.0, (n, d))).astype(dtype)
    idx, dist = P.nearest(pts, cent)
    ri, rd = _ref(pts, cent)
    np.testing.assert_array_equal(idx, ri)
    np.testing.assert_array_equal(dist, rd)


def test_nearest_ties_lowest_index_and_device_arrays():
    import torch

    rng = np.random.default_rng(3)
    cent = rng.integers(0, 4, (512, 16)).astype(np.float32)   # integer grid: many exact ties / duplicates
    cent[100] = cent[7]
    cent[300] = cent[7]
    pts = rng.integers(0, 4, (4000, 16)).astype(np.float32)
    pts[:50] = cent[300]
    ri, rd = _ref(pts, cent)
    idx, dist = P.nearest(pts, cent)
    np.testing.assert_array_equal(idx, ri)
    np.testing.assert_array_equal(dist, rd)
    assert (idx[:50] == 7).all()
    ti, td = P.nearest(torch.from_numpy(pts).cuda(), torch.from_numpy(cent).cuda())
    np.testing.assert_array_equal(ti.cpu().numpy(), ri)
    np.testing.assert_array_equal(td.cpu().numpy(), rd)


def test_nearest_argument_errors():
    with pytest.raises(ValueError):
        P.nearest(np.zeros((4, 8), np.float32), np.zeros((3, 9), np.float32))
