"""Multi-rank (N > 1) logic on CPU with gloo, world_size 2 (and an uneven 3).

Covers what the GPU path does across ranks: the z-slab partition (pure function in
the C-ABI, mirrored in Python), complete and disjoint coverage of every cascade,
and the in-place slab all-gather giving every rank the identical full atlas —
the same broadcast-per-slab exchange sdfgi_probes_update issues with NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_14394_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("res", [(32, 16, 32), (8, 8, 8), (12, 7, 9), (3, 2, 1)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_slabs_cover_each_probe_once_and_match_abi(res, world):
    n = res[0] * res[1] * res[2]
    owner = np.full(n, -1)
    for r in range(world):
        lo, hi = sharding.slab_range(res, r, world)
        assert (lo, hi) == sharding.slab_range_abi(res, r, world)
        assert np.all(owner[lo:hi] == -1)
        owner[lo:hi] = r
        assert lo % (res[0] * res[1]) == 0  # whole z-layers: one contiguous byte range of the atlas
    assert np.all(owner >= 0)


def _worker(rank, world, port, res, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = res[0] * res[1] * res[2]
    atlas = np.full((n, 10, 10, 3), -1.0, np.float32)
    lo, hi = sharding.slab_range(res, rank, world)
    # each rank "updates" its slab: tile value = probe index + 0.5 (deterministic)
    atlas[lo:hi] = (np.arange(lo, hi, dtype=np.float32) + 0.5)[:, None, None, None]
    sharding.allgather_slabs(atlas, res, dist)
    out[rank] = float(atlas.sum())
    expect = (np.arange(n, dtype=np.float64) + 0.5).sum() * 300
    assert np.allclose(atlas[:, 0, 0, 0], np.arange(n) + 0.5)
    assert abs(out[rank] - expect) < 1e-3 * expect
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,res", [(2, (8, 4, 8)), (3, (5, 3, 7))])
def test_slab_allgather_gloo(world, res):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, res, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert len(set(out.values())) == 1
