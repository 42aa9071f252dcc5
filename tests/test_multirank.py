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


def _worker(rank, world, port, out):
    """One rank of the sharded probe stage, with the oracle as the per-rank update:
    relocation replicated, the rank's z-slab (from the C-ABI's own partition)
    updated, the back-atlas slabs exchanged in place (one broadcast per slab, as
    sdfgi_probes_update does with NCCL), the other slabs' probes marked updated (as
    k_mark_updated does on the device)."""
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py
    from golden_util import load

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = load("c1")
    res = case.res
    n = res[0] * res[1] * res[2]
    ora = oracle_py.Stage(case.scene, cfg=case.cfg(), res=res, spacing=case.spacing)
    lo, hi = sharding.slab_range_abi(res, rank, world)
    mine = np.array([[0, i] for i in range(lo, hi)], np.int32).reshape(-1, 2)
    others = np.array([[0, i] for i in range(n) if not lo <= i < hi], np.int32).reshape(-1, 2)
    for p in range(len(case.passes)):
        ora.relocate_all()
        ora.update_refs(p, mine)
        atlas = ora.atlas(0)
        sharding.allgather_slabs(atlas, res, dist)
        ora.set_atlas(0, atlas)
        ora.mark_updated(p, others)
    out[rank] = (ora.atlas(0).tobytes(), ora.probes(0).tobytes())
    dist.barrier()
    dist.destroy_process_group()


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_probe_stage_gloo_equals_single_rank(world):
    """SURVEY §8e's correctness test on CPU: Cornell C1, all of its golden passes,
    on `world` gloo ranks (z-slabs of 8 layers: 4+4, 2+3+3) — every rank ends with
    the atlas and probe states of the single-rank run, bit for bit, and those are
    the reference's own (golden) outputs."""
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_util import load

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert len(out) == world and len(set(out.values())) == 1
    case = load("c1")
    last = len(case.passes) - 1
    atlas = np.frombuffer(out[0][0], np.float32)
    assert np.array_equal(atlas, case.data[f"atlas_p{last}_c0"].astype(np.float32).ravel())
