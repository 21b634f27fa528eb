"""GPU: the sharded exchange over NCCL on one device (world size 1): the
packed single all-gather round-trips distances, ids and counts, and the device
merge of G copies of one result list returns that list (the exchange used by
bench.py --gpus N > 1)."""

import os
import socket

import numpy as np
import pytest

import paper_1712_02912_b200 as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_packed_all_gather_and_merge(nccl_group):
    import torch

    from paper_1712_02912_b200.sharded import all_gather_results

    rng = np.random.default_rng(4)
    nq, r = 7, 33
    d = torch.from_numpy(np.sort(rng.uniform(0, 100, (nq, r)), axis=1)).cuda()
    i = torch.from_numpy(rng.integers(0, 10**9, (nq, r))).cuda()
    c = torch.from_numpy(rng.integers(0, r + 1, nq).astype(np.int32)).cuda()
    gd, gi, gc = all_gather_results(d, i, c)
    assert gd.shape == (1, nq, r) and gd.dtype == torch.float64 and gc.dtype == torch.int32
    assert torch.equal(gd[0], d) and torch.equal(gi[0], i) and torch.equal(gc[0], c)
    # merge with a second shard holding the same distances under other ids:
    # the top-r of the union by (distance, id)
    off = 10**10
    md, mi, mc = P.merge_topr(torch.cat([gd, gd]), torch.cat([gi, gi + off]), torch.cat([gc, gc]), r)
    md, mi, mc = md.cpu().numpy(), mi.cpu().numpy(), mc.cpu().numpy()
    dn, inn, cn = d.cpu().numpy(), i.cpu().numpy(), c.cpu().numpy()
    for q in range(nq):
        own = list(zip(dn[q, :cn[q]], inn[q, :cn[q]]))
        pairs = sorted(own + [(a, b + off) for a, b in own])[:r]
        assert mc[q] == len(pairs)
        assert [(a, b) for a, b in zip(md[q, :mc[q]], mi[q, :mc[q]])] == pairs
