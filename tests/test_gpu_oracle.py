"""GPU vs the C oracle on the bench workload (C2: ~2k primitives, 275 clusters,
32x16x32 probes, 256 rays).

The oracle is bit-exact with the reference (test_oracle.py), so it stands in for
the reference at sizes the golden fixtures do not cover. Full-size checks use
size-independent properties: bit-exact relocation of the whole volume, bit-exact
SDF queries, run-to-run determinism, non-negative texels. Ray-level parity runs
on a probe sample the oracle finishes in seconds.
"""
import os
import sys

import numpy as np
import pytest

from paper_2007_14394_b200 import api, scene_io
from paper_2007_14394_b200.runtime import Device

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py  # noqa: E402

pytestmark = pytest.mark.gpu

C2 = os.path.join(ROOT, "paper_2007_14394_b200", "data", "c2.sdfs")


@pytest.fixture(scope="module")
def scene():
    return scene_io.read_sdfs(C2)


@pytest.fixture(scope="module")
def dev():
    d = Device(0, precision="f64")
    yield d
    d.close()


def rel_err(got, want):
    floor = 0.05 * max(float(np.mean(np.abs(want))), 1e-12)
    return np.abs(got.astype(np.float64) - want) / np.maximum(np.abs(want), floor)


@pytest.mark.parametrize("accel", [0, 1], ids=["flatwalk", "grid"])
def test_c2_queries_bit_exact(dev, scene, accel):
    """querySceneSdf values AND owners identical to the reference walk, including
    points off the candidate grid (supercluster path) and seeded queries."""
    dev.upload_scene(scene)
    dev.set_accel(accel)
    ora = oracle_py.Stage(scene)
    rng = np.random.default_rng(5)
    pts = np.concatenate([rng.uniform([-7.5, -1, -5.5], [7.5, 7.5, 5.5], size=(20000, 3)),
                          rng.uniform([-40, -5, -40], [40, 40, 40], size=(2000, 3))])
    d_g, o_g = dev.query_points(pts)
    d_o, o_o = ora.query(pts)
    assert np.array_equal(d_g, d_o)
    assert np.array_equal(o_g, o_o)
    init = np.abs(d_o) * rng.uniform(0.2, 3.0, len(pts))
    d_g, o_g = dev.query_points(pts, init)
    d_o, o_o = ora.query(pts, init)
    assert np.array_equal(d_g, d_o) and np.array_equal(o_g, o_o)
    dev.set_accel(1)


def test_c2_relocation_bit_exact_full_volume(dev, scene):
    stage = api.ProbeStage(dev, scene)
    ora = oracle_py.Stage(scene)
    for p in range(2):
        rep = stage.relocate_all()[0]
        orep, _ = ora.relocate_all()
        assert [int(rep["relocated"]), int(rep["rejected"]), int(rep["dead"])] == list(orep[0])
        g, o = dev.probes(0), ora.probes(0)
        for f in ("pos", "last_pos", "alive", "reject_history"):
            assert np.array_equal(g[f], o[f]), f
        # mark updated as the update would, without tracing: pass-through frame
        res = api.updateProbes(dev, stage.cfg, p, refs=np.zeros((0, 2), np.int32))
        assert int(res["rays_traced"]) == 0
        dev.swap()


def test_c2_sampled_update_matches_oracle(dev, scene):
    """Every 128th probe of the C2 volume through 2 bounces: identical probe states,
    identical ray counts, texels within the 1e-3 bar (FP64; bit-identical except
    where direction ulps flip a corner-tie owner)."""
    stride = 128
    stage = api.ProbeStage(dev, scene)
    ora = oracle_py.Stage(scene)
    n = 32 * 16 * 32
    refs = np.array([[0, i] for i in range(0, n, stride)], np.int32)
    for p in range(2):
        stage.relocate_all()
        res = api.updateProbes(dev, stage.cfg, p, refs=refs)
        dev.swap()
        _, _, (md, rays, upd, _) = ora.run_pass(p, stride=stride, threads=os.cpu_count() or 1)
        assert int(res["rays_traced"]) == rays and int(res["probes_updated"]) == upd
        g, o = dev.probes(0), ora.probes(0)
        for f in ("pos", "alive", "reject_history", "last_update_frame"):
            assert np.array_equal(g[f], o[f]), (p, f)
        ga, oa = dev.atlas(0), ora.atlas(0)
        err = rel_err(ga, oa)
        assert np.mean(err > 1e-3) <= 1e-3 and err.max() <= 1e-2, (p, err.max())
        assert np.mean(ga == oa) > 0.99, p


def test_c2_full_frame_deterministic_and_non_negative(dev, scene):
    """Two full 3-bounce C2 frames are bit-identical run to run (fixed-order
    reductions, no float atomics), and every texel is >= 0 (test_probe_update.cpp:263-278)."""
    out = []
    for _ in range(2):
        stage = api.ProbeStage(dev, scene)
        for p in range(3):
            stage.run_pass(p)
        out.append(dev.atlas(0))
    assert np.array_equal(out[0], out[1])
    assert np.all(out[0] >= 0) and np.all(np.isfinite(out[0]))


def test_c2_f32_mode_error_report(scene):
    """FP32 perf mode against the oracle on sampled probes: the north-star 1e-3 bar
    holds for nearly every channel; the tail comes from hit/miss and owner flips."""
    stride = 128
    with Device(0, precision="f32") as d32:
        stage = api.ProbeStage(d32, scene)
        ora = oracle_py.Stage(scene)
        n = 32 * 16 * 32
        refs = np.array([[0, i] for i in range(0, n, stride)], np.int32)
        stage.relocate_all()
        api.updateProbes(d32, stage.cfg, 0, refs=refs)
        d32.swap()
        ora.run_pass(0, stride=stride, threads=os.cpu_count() or 1)
        err = rel_err(d32.atlas(0)[::stride], ora.atlas(0)[::stride])
        frac = float(np.mean(err > 1e-3))
        print(f"FP32 C2 texels: max rel err {err.max():.3e}, {frac:.2e} of channels over 1e-3")
        assert frac < 2e-2
