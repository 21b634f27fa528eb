"""Full-size parity (tests/parity_full.py): every query of cfg0/1/2 (1,000)
and cfg3 (10,000 at Q = 10,000), and cfg4 as 8 x 125M shards (sharded ==
unsharded for all 10,000 queries; a seeded 64-query sample against the oracle
over all 1e9 codes).  Zero mismatches in ids and distances / bins."""

import pytest

from tests import parity_full as F

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", ["cfg0", "cfg1", "cfg2"])
def test_exhaustive_all_queries(name):
    res = F.exhaustive(name)
    assert res["queries_checked"] == res["queries_in_batch"] == 1000
    assert res["mismatches"] == 0, res["mismatched_queries"][:20]


def test_ivf_all_queries():
    res = F.ivf()
    assert res["queries_checked"] == res["queries_in_batch"] == 10_000
    assert res["mismatches"] == 0, res["mismatched_queries"][:20]


def test_billion_sharded_and_oracle_sample():
    res = F.billion()
    assert res["codes"] == 1_000_000_000 and res["shards"] == 8
    assert res["sharded_vs_unsharded"]["queries_checked"] == 10_000
    assert res["sharded_vs_unsharded"]["mismatches"] == 0, res["sharded_vs_unsharded"]["mismatched_queries"]
    assert res["oracle"]["queries_checked"] >= 64
    assert res["oracle"]["mismatches"] == 0, res["oracle"]["mismatched_queries"]
