"""GPU, world size 2: two processes each run the DEVICE sharded search on
cuda:0 (their own shard of one global list / their own greedy share of the
inverted lists) and exchange through gloo on host tensors -- no kernel waits
on another rank.  The merged results equal the CPU oracle's unsharded answer
(scan.py:197-203, quickadc.py:104-141 with the global prefix, ivf.py:148-196);
`search_stream` (exchange of batch i overlapped with the scan of batch i+1)
returns the same as per-batch `search`."""

import os
import socket
import tempfile

import numpy as np
import pytest

from oracle import pqscan_oracle as O
from tests.helpers import encode, kmeans_books, mixture

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(71)
    x = mixture(rng, 120_000, 32, comps=32)
    books4 = kmeans_books(x[:6000], 8, 16, iters=3)
    books8 = kmeans_books(x[:6000], 4, 256, iters=2)
    qs = x[:24] + 0.7
    coarse = x[rng.choice(len(x), 64, replace=False)].copy()
    return x, books4, books8, qs, coarse


def _ivf_arrays(x, books8, coarse):
    cells = ((x[:, None, :] - coarse[None]) ** 2).sum(-1).argmin(1)
    order = np.argsort(cells, kind="stable")
    res = (x.astype(np.float64) - coarse[cells].astype(np.float64)).astype(np.float32)
    codes = O.encode(books8, res[order].astype(np.float64))
    sizes = np.bincount(cells, minlength=coarse.shape[0]).astype(np.int64)
    return sizes, codes, order.astype(np.int64)


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    import paper_1712_02912_b200 as P
    from paper_1712_02912_b200.sharded import ShardedSearch, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, books4, books8, qs, coarse = _data()
    n = x.shape[0]
    lo, hi = shard_range(n, world, rank)
    qd = torch.from_numpy(qs).cuda()
    out = {}
    # Quick ADC, global prefix
    codes4 = encode(books4, x)
    pq4 = P.ProductQuantizer(8, 4, 32, books4)
    s4 = ShardedSearch.quick_adc(codes4[lo:hi], rank, world, n, codes4[:200], pq4, 200)
    d, i, c = s4.search(qd, 50)
    out["q_d"], out["q_i"], out["q_c"] = d.cpu().numpy(), i.cpu().numpy(), c.cpu().numpy()
    # float ADC
    codes8 = encode(books8, x)
    pq8 = P.ProductQuantizer(4, 8, 32, books8)
    s8 = ShardedSearch.float_adc(codes8[lo:hi], rank, world, n, pq8)
    d, i, c = s8.search(qd, 40)
    out["f_d"], out["f_i"], out["f_c"] = d.cpu().numpy(), i.cpu().numpy(), c.cpu().numpy()
    # IVF, lists partitioned; stream of two batches
    sizes, ivf_codes, ivf_ids = _ivf_arrays(x, books8, coarse)
    si = ShardedSearch.ivf(pq8, coarse, sizes, ivf_codes, ivf_ids, rank, world, ma=6)
    res = list(si.search_stream([qd[:12], qd[12:]], 30))
    out["v_d"] = np.concatenate([r[0].cpu().numpy() for r in res])
    out["v_i"] = np.concatenate([r[1].cpu().numpy() for r in res])
    out["v_c"] = np.concatenate([r[2].cpu().numpy() for r in res])
    out["owned"] = np.array([int((si.owner == rank).sum())])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_device_search_equals_oracle():
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(2, _port(), td), nprocs=2, join=True)
        r0 = dict(np.load(os.path.join(td, "rank0.npz")))
        r1 = dict(np.load(os.path.join(td, "rank1.npz")))
    for k in r0:
        if k != "owned":
            np.testing.assert_array_equal(r0[k], r1[k])   # every rank holds the merged answer
    assert r0["owned"][0] + r1["owned"][0] == 64 and min(r0["owned"][0], r1["owned"][0]) > 0
    x, books4, books8, qs, coarse = _data()
    ids = np.arange(x.shape[0], dtype=np.int64)
    codes4, codes8 = encode(books4, x), encode(books8, x)
    sizes, ivf_codes, ivf_ids = _ivf_arrays(x, books8, coarse)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    lc = [ivf_codes[offs[k]:offs[k + 1]] for k in range(64)]
    li = [ivf_ids[offs[k]:offs[k + 1]] for k in range(64)]
    for qi, q in enumerate(qs):
        b, i, _, _, _ = O.qadc_scan(codes4, ids, O.compute_tables(books4, q), 200, 50)
        np.testing.assert_array_equal(r0["q_d"][qi][:len(b)], b)
        np.testing.assert_array_equal(r0["q_i"][qi][:len(i)], i)
        d, i = O.scan(codes8, ids, O.compute_tables(books8, q), 40)
        np.testing.assert_array_equal(r0["f_d"][qi], d)
        np.testing.assert_array_equal(r0["f_i"][qi], i)
        d, i = O.query_ivf(coarse, books8, lc, li, q, 6, 30)
        assert r0["v_c"][qi] == len(d)
        np.testing.assert_array_equal(r0["v_d"][qi][:len(d)], d)
        np.testing.assert_array_equal(r0["v_i"][qi][:len(i)], i)
