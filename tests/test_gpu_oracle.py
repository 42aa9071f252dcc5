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


def test_c2_full_step_matches_oracle(dev, scene, oracle_c2):
    """The bench workload itself, every probe of the 32x16x32 volume through all 3
    bounces (15M rays) against the oracle: relocation reports and probe states
    bit-exact; every texel channel within the north-star 1e-3 relative. Measured:
    every texel of all three bounces bit-identical to the oracle (the MVC sines are
    evaluated algebraically, a few FP64 ulps, which the float texels absorb)."""
    stage = api.ProbeStage(dev, scene)
    for p, want in enumerate(oracle_c2["passes"]):
        rep = stage.relocate_all()[0]
        assert [int(rep["relocated"]), int(rep["rejected"]), int(rep["dead"])] == want["rep"], p
        res = api.updateProbes(dev, stage.cfg, p)
        dev.swap()
        assert int(res["rays_traced"]) == want["rays"] and int(res["probes_updated"]) == want["upd"], p
        g, o = dev.probes(0), want["probes"]
        for f in ("pos", "last_pos", "alive", "reject_history", "last_update_frame"):
            assert np.array_equal(g[f], o[f]), (p, f)
        ga, oa = dev.atlas(0), want["atlas"]
        err = rel_err(ga, oa)
        print(f"C2 pass {p}: max texel rel err {err.max():.3e}, bit-identical {np.mean(ga == oa):.6f}")
        assert err.max() <= 1e-3, (p, err.max())
        assert np.mean(ga == oa) > 0.9999, p


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


def test_c2_f32_mode_error_report(scene, oracle_c2):
    """FP32 perf mode against the oracle on the whole C2 step (every probe, 3
    bounces): the error distribution is reported; the tail comes from hit/miss and
    owner flips of float traces."""
    with Device(0, precision="f32") as d32:
        stage = api.ProbeStage(d32, scene)
        for p, want in enumerate(oracle_c2["passes"]):
            stage.run_pass(p)
            err = rel_err(d32.atlas(0), want["atlas"])
            frac = float(np.mean(err > 1e-3))
            print(f"FP32 C2 pass {p}: max rel err {err.max():.3e}, p99.9 {np.quantile(err, 0.999):.3e}, "
                  f"{frac:.2e} of channels over 1e-3")
            assert frac < 2e-2
