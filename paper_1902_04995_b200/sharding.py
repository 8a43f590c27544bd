"""LP-index sharding across GPUs / ranks.

LPs are independent, so a multi-GPU solve is a partition of the LP index
range with no data-path collective. Seeds are keyed by GLOBAL LP index
(lp2dgen_fill's `first`), so any partition reproduces the single-GPU batch.
"""
from __future__ import annotations

import numpy as np

from . import _native as N


def partition(m, parts: int) -> np.ndarray:
    """Contiguous ranges balanced by sum(m + 4): cut[g]..cut[g+1] (C ABI
    lp2dgpu_partition, the same routine host-mode solves use)."""
    m = np.ascontiguousarray(m, dtype=np.int32)
    cut = np.zeros(parts + 1, np.int64)
    rc = N.lib().lp2dgpu_partition(len(m), m.ctypes.data, parts, cut.ctypes.data)
    if rc:
        raise ValueError(N.last_error())
    return cut


def shard_of(m_global, rank: int, world: int):
    cut = partition(m_global, world)
    return int(cut[rank]), int(cut[rank + 1])


def generate_shard(m_global, seed: int, rank: int, world: int, **kw):
    """The rank's slice of PackedBatch.generate(m_global, seed)."""
    from .lp2d import PackedBatch

    lo, hi = shard_of(m_global, rank, world)
    return lo, PackedBatch.generate(np.asarray(m_global)[lo:hi], seed, first=lo, **kw)
