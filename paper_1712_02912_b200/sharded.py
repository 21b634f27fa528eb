"""Database sharding across GPUs: one process per GPU.

Each rank owns a contiguous id range of one global code list and scans the
whole query batch; the per-rank top-r lists are all-gathered with
torch.distributed (NCCL over NVLink between GPUs; gloo works for CPU tests)
and merged on the device by `pqs_merge_topr` -- the reference's
NeighborSet.push merge (scan.py:109-118), exact because the global top-r is a
subset of the union of the shard top-r under the same (distance, id) order.

Quick ADC needs *global* quantization parameters: qmax is the r-th fp64 ADC
of the first init_count codes of the global list (quickadc.py:130-137), so
those codes are replicated to every rank (`prefix_codes`).

IVFADC shards the inverted lists: every rank holds the coarse
quantizer and the residual codebooks (the probes are computed identically
everywhere) but only its own lists -- assigned greedily by length, largest
first, to the least-loaded rank -- and returns the exact top-r over the
probed lists it owns; the same all-gather + (distance, id) merge gives the
reference's query_ivf result (ivf.py:174-195 merges per-list top-r the same
way).

`search_stream` overlaps the exchange of one query batch with the scan of the
next: the all-gather is issued asynchronously, the next batch's scan is
queued on the compute stream, and only then is the previous batch merged.
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced id range [lo, hi) of `rank` among `world` shards."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def all_gather_results(dist, ids, cnt, group=None):
    """Gather (G, nq, r) dist/ids and (G, nq) counts from every rank with ONE
    collective: each rank packs [fp64 distance bits | ids | count] into an
    (nq, 2r + 1) int64 block (the per-step exchange is latency-, not
    bandwidth-bound, so one all-gather instead of three)."""
    _, finish = all_gather_start(dist, ids, cnt, group)
    return finish()


def all_gather_start(dist, ids, cnt, group=None):
    """Issue the packed all-gather asynchronously; returns (handle, finish)
    where finish() waits and unpacks (gd, gi, gc).  CUDA tensors on a gloo
    group (CPU tests of the device path) are staged through host memory."""
    import torch
    import torch.distributed as dist_

    world = dist_.get_world_size(group)
    dist, ids, cnt = (torch.from_numpy(np.ascontiguousarray(t)) if isinstance(t, np.ndarray) else t
                      for t in (dist, ids, cnt))
    nq, r = dist.shape
    packed = torch.cat([dist.to(torch.float64).contiguous().view(torch.int64), ids.to(torch.int64),
                        cnt.to(torch.int64).reshape(nq, 1)], dim=1).contiguous()
    dev = packed.device
    if packed.is_cuda and dist_.get_backend(group) == "gloo":
        packed = packed.cpu()
    out = torch.empty((world * nq, packed.shape[1]), dtype=torch.int64, device=packed.device)
    work = dist_.all_gather_into_tensor(out, packed, group=group, async_op=True)  # rank blocks along dim 0

    def finish():
        work.wait()
        return _unpack(out.to(dev), world, nq, r, cnt.dtype)

    return work, finish


def _unpack(out, world, nq, r, cnt_dtype):
    out = out.view(world, nq, 2 * r + 1)
    import torch

    gd = out[:, :, :r].contiguous().view(torch.float64)
    gi = out[:, :, r:2 * r].contiguous()
    gc = out[:, :, 2 * r].to(cnt_dtype).contiguous()
    return gd, gi, gc


def partition_lists(sizes, world: int):
    """Greedy list partition: lists in decreasing size order, each
    to the rank with the smallest total so far (ties: lowest rank, then the
    lower list index first).  Returns owner (K,) int64."""
    sizes = np.asarray(sizes, dtype=np.int64)
    if world < 1:
        raise ValueError("bad world")
    order = np.argsort(-sizes, kind="stable")
    load = np.zeros(world, dtype=np.int64)
    owner = np.empty(sizes.shape[0], dtype=np.int64)
    import heapq

    heap = [(0, g) for g in range(world)]
    for c in order:
        ld, g = heapq.heappop(heap)
        owner[c] = g
        load[g] = ld + int(sizes[c])
        heapq.heappush(heap, (int(load[g]), g))
    return owner


class ShardedSearch:
    """One rank's shard of a global list plus the exchange + merge step.

    local_search(queries, r) -> (dist float64 (nq, r), ids int64 (nq, r),
    count int32 (nq,)) with GLOBAL ids; merge(dist, ids, cnt, r) merges the
    gathered (G, nq, r) lists.  Both default to the device engine; tests
    inject oracle-backed callables to check the host logic on CPU (gloo).
    """

    def __init__(self, local_search: Callable, merge: Callable | None = None, group=None):
        self.local_search = local_search
        self.merge = merge
        self.group = group

    @classmethod
    def quick_adc(cls, codes_local, rank: int, world: int, n_total: int, prefix_codes, pq, init_count: int,
                  ctx=None, group=None):
        """Device-backed Quick ADC shard (ids = global offset + local index)."""
        import torch

        from .engine import DeviceCodes, DeviceQuantizer, merge_topr

        lo, hi = shard_range(n_total, world, rank)
        if codes_local.shape[0] != hi - lo:
            raise ValueError("codes_local does not match this rank's shard")
        db = DeviceCodes(codes_local, 4, id_base=lo, ctx=ctx)
        db.set_prefix(prefix_codes)
        dq = DeviceQuantizer(pq, ctx)

        def local(queries, r):
            bins, ids, cnt, _, _ = db.qadc_search(dq, queries, init_count, r)
            return bins.to(torch.float64), ids, cnt

        def merge(d, i, c, r):
            return merge_topr(d, i, c, r, ctx=ctx)

        out = cls(local, merge, group)
        out.db, out.dq = db, dq
        return out

    @classmethod
    def float_adc(cls, codes_local, rank: int, world: int, n_total: int, pq, ctx=None, group=None):
        from .engine import DeviceCodes, DeviceQuantizer, merge_topr

        lo, hi = shard_range(n_total, world, rank)
        if codes_local.shape[0] != hi - lo:
            raise ValueError("codes_local does not match this rank's shard")
        db = DeviceCodes(codes_local, 8, id_base=lo, ctx=ctx)
        dq = DeviceQuantizer(pq, ctx)

        def local(queries, r):
            return db.adc_search(dq, queries, r)

        out = cls(local, lambda d, i, c, r: merge_topr(d, i, c, r, ctx=ctx), group)
        out.db, out.dq = db, dq
        return out

    @classmethod
    def ivf(cls, pq, coarse, list_sizes, codes, ids, rank: int, world: int, ma: int, ctx=None, group=None):
        """Device-backed IVF shard: this rank's lists of an index given in
        cell order (list_sizes host (K,), codes (n, m), ids (n,) -- numpy or
        CUDA tensors); the other lists are empty here."""
        import torch

        from .engine import DeviceIvf, merge_topr

        sizes = np.asarray(list_sizes, dtype=np.int64)
        owner = partition_lists(sizes, world)
        mine = owner == rank
        local_sizes = np.where(mine, sizes, 0)
        if isinstance(codes, np.ndarray):
            keep = np.repeat(mine, sizes)
            lc, li = np.ascontiguousarray(codes[keep]), np.ascontiguousarray(ids[keep])
        else:
            keep = torch.from_numpy(np.repeat(mine, sizes)).to(codes.device)
            lc, li = codes[keep].contiguous(), ids[keep].contiguous()
        div = DeviceIvf.from_arrays(pq, coarse, local_sizes, lc, li, ctx=ctx)

        def local(queries, r):
            return div.search(queries, ma, r)

        out = cls(local, lambda d, i, c, r: merge_topr(d, i, c, r, ctx=ctx), group)
        out.ivf_index, out.owner = div, owner
        return out

    def search_stream(self, batches, r: int):
        """Global top-r for each query batch of an iterable, the exchange of
        batch i overlapping the scan of batch i+1 (yields (dist, ids, count)
        per batch, in order)."""
        import torch.distributed as dist_

        multi = dist_.is_available() and dist_.is_initialized() and dist_.get_world_size(self.group) > 1
        pending = None
        for q in batches:
            d, i, c = self.local_search(q, r)            # queued on the compute stream
            if not multi:
                yield d, i, c
                continue
            _, fin = all_gather_start(d, i, c, self.group)
            if pending is not None:
                gd, gi, gc = pending()
                yield self.merge(gd, gi, gc, r)
            pending = fin
        if pending is not None:
            gd, gi, gc = pending()
            yield self.merge(gd, gi, gc, r)

    def search(self, queries, r: int):
        """Global top-r for every query (identical result on every rank)."""
        import torch.distributed as dist_

        d, i, c = self.local_search(queries, r)
        if not dist_.is_available() or not dist_.is_initialized() or dist_.get_world_size(self.group) == 1:
            return d, i, c
        gd, gi, gc = all_gather_results(d, i, c, self.group)
        return self.merge(gd, gi, gc, r)


__all__ = ["shard_range", "partition_lists", "all_gather_results", "all_gather_start", "ShardedSearch"]
