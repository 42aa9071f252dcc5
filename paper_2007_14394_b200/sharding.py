"""Probe-slab sharding across ranks, host side.

The device path (sdfgi_probes_update with world > 1) traces only the rank's z-slab
and exchanges the back-atlas slabs in place with one broadcast per slab (NCCL).
This module holds the same partition as a pure function plus the exchange
pattern over torch.distributed, so the multi-rank logic is testable on CPU with
gloo (tests/test_multirank.py) and usable for host-side atlas copies.
"""
from __future__ import annotations

import ctypes

import numpy as np


def slab_range(res, rank, world):
    """Probe-index range [lo, hi) owned by `rank` (== sdfgi_slab_range)."""
    rx, ry, rz = (int(r) for r in res)
    z0 = (rz * rank) // world
    z1 = (rz * (rank + 1)) // world
    return z0 * rx * ry, z1 * rx * ry


def slab_range_abi(res, rank, world):
    """The C-ABI's partition (no device needed)."""
    from .runtime import _call

    lo, hi = ctypes.c_int(), ctypes.c_int()
    _call("sdfgi_slab_range", int(res[0]), int(res[1]), int(res[2]), rank, world, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def allgather_slabs(atlas: np.ndarray, res, dist, group=None):
    """In-place all-gather of per-rank probe slabs of a [P, T, T, 3] float atlas:
    one broadcast per slab from its owner, as the device path does with
    ncclBroadcast inside one group. Works with any torch.distributed backend."""
    import torch

    world = dist.get_world_size(group)
    t = torch.from_numpy(atlas)
    for r in range(world):
        lo, hi = slab_range(res, r, world)
        if hi <= lo:
            continue
        view = t[lo:hi].contiguous()
        dist.broadcast(view, src=r, group=group)
        t[lo:hi] = view
    return atlas
