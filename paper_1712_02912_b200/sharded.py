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
    import torch
    import torch.distributed as dist_

    world = dist_.get_world_size(group)
    nq, r = dist.shape
    packed = torch.cat([dist.to(torch.float64).contiguous().view(torch.int64), ids.to(torch.int64),
                        cnt.to(torch.int64).reshape(nq, 1)], dim=1).contiguous()
    out = torch.empty((world * nq, packed.shape[1]), dtype=torch.int64, device=packed.device)
    dist_.all_gather_into_tensor(out, packed, group=group)  # rank blocks concatenated along dim 0
    out = out.view(world, nq, packed.shape[1])
    gd = out[:, :, :r].contiguous().view(torch.float64)
    gi = out[:, :, r:2 * r].contiguous()
    gc = out[:, :, 2 * r].to(cnt.dtype).contiguous()
    return gd, gi, gc


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

    def search(self, queries, r: int):
        """Global top-r for every query (identical result on every rank)."""
        import torch.distributed as dist_

        d, i, c = self.local_search(queries, r)
        if not dist_.is_available() or not dist_.is_initialized() or dist_.get_world_size(self.group) == 1:
            return d, i, c
        gd, gi, gc = all_gather_results(d, i, c, self.group)
        return self.merge(gd, gi, gc, r)


__all__ = ["shard_range", "all_gather_results", "ShardedSearch"]
