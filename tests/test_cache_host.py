"""CPU-only: device-cache coherence logic of the drop-in containers
(paper_1712_02912_b200/_cache.py, types._Sealable): uploaded arrays become
read-only, rebinding a field or changing IvfIndex.lists bumps the mutation
epoch, and the cache rebuilds exactly then."""

import numpy as np
import pytest

import paper_1712_02912_b200 as P
from paper_1712_02912_b200._cache import device_cached
from paper_1712_02912_b200.types import implicit_ids, mutation_epoch


def test_cache_rebuilds_on_rebinding_only():
    cl = P.CodeList(np.zeros((10, 4), np.uint8))
    builds = []

    def get():
        return device_cached(cl, "_t", (cl.codes, cl.ids), lambda: builds.append(1) or len(builds))

    assert get() == 1 and get() == 1
    with pytest.raises(ValueError):
        cl.codes[0, 0] = 1                      # frozen by the upload
    cl.codes = np.ones((10, 4), np.uint8)       # rebinding
    assert get() == 2 and get() == 2
    e = mutation_epoch()
    P.CodeList(np.zeros((3, 4), np.uint8))      # constructing others does not invalidate
    assert mutation_epoch() == e and get() == 2


def test_implicit_ids_follow_the_array():
    cl = P.CodeList(np.zeros((5, 2), np.uint8))
    assert implicit_ids(cl)
    cl.ids = np.arange(5, dtype=np.int64)       # equal values, but a user array: explicit
    assert not implicit_ids(cl)
    tl = P.transpose_blocks(P.CodeList(np.zeros((5, 2), np.uint8)), 4)
    assert implicit_ids(tl)


def test_ivf_lists_are_tracked():
    pq = P.ProductQuantizer(2, 4, 4, np.zeros((2, 16, 2), np.float32))
    idx = P.IvfIndex(np.zeros((2, 4), np.float32), pq, [P.CodeList(np.zeros((1, 2), np.uint8)) for _ in range(2)])
    e = mutation_epoch()
    idx.lists[1] = P.CodeList(np.zeros((2, 2), np.uint8))
    assert mutation_epoch() > e
    e = mutation_epoch()
    idx.lists = [P.CodeList(np.zeros((1, 2), np.uint8))] * 2   # rebinding wraps the new list too
    assert mutation_epoch() > e
    e = mutation_epoch()
    idx.lists.append(P.CodeList(np.zeros((1, 2), np.uint8)))
    assert mutation_epoch() > e
