"""Device copies of the drop-in's host containers, cached on the containers.

The reference recomputes from its arrays on every call; the GPU drop-in
uploads them once.  A cache entry is keyed on the identity of the arrays it
uploaded (the entry keeps them alive, so ids are never reused) and on the
global mutation epoch (types.mutation_epoch: bumped when a field of a sealed
container is rebound or an IvfIndex's list of lists is changed), and every
uploaded array is made read-only -- an in-place edit afterwards raises
instead of silently searching stale device data.
"""

from __future__ import annotations

import numpy as np

from .types import mutation_epoch


def freeze(a):
    if isinstance(a, np.ndarray) and a.flags.writeable:
        a.flags.writeable = False
    return a


def device_cached(obj, slot: str, arrays, build):
    """build() once per (epoch, array identities, other key values); arrays are frozen first."""
    key = (mutation_epoch(),) + tuple(
        (id(a), a.__array_interface__["data"][0], a.shape, a.dtype.str) if isinstance(a, np.ndarray) else ("v", a)
        for a in arrays)
    ent = obj.__dict__.get(slot)
    if ent is None or ent[0] != key:
        for a in arrays:
            freeze(a)
        ent = (key, tuple(arrays), build())
        object.__setattr__(obj, slot, ent)
    return ent[2]
