"""CPU, world_size 2 over gloo: the sharded search's host logic (shard ranges,
global ids, global Quick ADC prefix, all-gather, merge) reproduces the
unsharded reference result.  The per-shard scan and the merge are the CPU
oracle here (the device versions are covered by the -m gpu tests)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pqscan_oracle as O
from paper_1712_02912_b200.sharded import ShardedSearch, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(11)
    books = rng.uniform(0, 10, (8, 16, 4)).astype(np.float32)
    codes = rng.integers(0, 16, (3001, 8)).astype(np.uint8)
    qs = rng.uniform(0, 10, (5, 32)).astype(np.float32)
    return books, codes, qs


def _shard_qadc(books, codes_local, lo, prefix, init, r):
    """Oracle per-shard Quick ADC with GLOBAL params (quickadc.py:129-141)."""

    def local(queries, rr):
        nq = queries.shape[0]
        d = np.full((nq, rr), np.inf)
        i = np.full((nq, rr), -1, np.int64)
        c = np.zeros(nq, np.int32)
        for qi, q in enumerate(queries.numpy()):
            t = O.compute_tables(books, q)
            qmin, qmax = O.qadc_params(t, prefix, init, rr)
            bins = O.quantized_distances(codes_local, O.quantize(qmin, qmax, t)).astype(np.float64)
            bd, bi = O.select_best(bins, np.arange(lo, lo + codes_local.shape[0], dtype=np.int64), rr)
            d[qi, :len(bd)], i[qi, :len(bi)], c[qi] = bd, bi, len(bd)
        return torch.from_numpy(d), torch.from_numpy(i), torch.from_numpy(c)

    return local


def _oracle_merge(gd, gi, gc, r):
    G, nq, _ = gd.shape
    d = np.full((nq, r), np.inf)
    i = np.full((nq, r), -1, np.int64)
    c = np.zeros(nq, np.int32)
    for q in range(nq):
        md, mi = O.merge_shards([gd[g, q, :gc[g, q]].numpy() for g in range(G)],
                                [gi[g, q, :gc[g, q]].numpy() for g in range(G)], r)
        d[q, :len(md)], i[q, :len(mi)], c[q] = md, mi, len(md)
    return d, i, c


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        books, codes, qs = _data()
        lo, hi = shard_range(codes.shape[0], world, rank)
        init, r = 200, 40
        prefix = codes[:min(init, codes.shape[0])]  # replicated global prefix
        s = ShardedSearch(_shard_qadc(books, codes[lo:hi], lo, prefix, init, r), _oracle_merge)
        d, i, c = s.search(torch.from_numpy(qs), r)
        out_q.put((rank, np.asarray(d), np.asarray(i), np.asarray(c)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_quick_adc_equals_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q)) for rk in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    books, codes, qs = _data()
    ids = np.arange(codes.shape[0], dtype=np.int64)
    for rank, d, i, c in res:
        for qi, qv in enumerate(qs):
            ob, oi, _, _, _ = O.qadc_scan(codes, ids, O.compute_tables(books, qv), 200, 40)
            assert c[qi] == len(ob)
            np.testing.assert_array_equal(d[qi, :c[qi]], ob)
            np.testing.assert_array_equal(i[qi, :c[qi]], oi)


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_partition_lists_greedy_balanced():
    from paper_1712_02912_b200.sharded import partition_lists

    rng = np.random.default_rng(3)
    sizes = rng.integers(0, 5000, 1000)
    for world in (1, 2, 3, 8):
        owner = partition_lists(sizes, world)
        assert owner.shape == sizes.shape and owner.min() >= 0 and owner.max() < world
        loads = np.bincount(owner, weights=sizes, minlength=world)
        assert loads.sum() == sizes.sum()
        assert loads.max() - loads.min() <= sizes.max()   # LPT bound
    assert (partition_lists(sizes, 1) == 0).all()
