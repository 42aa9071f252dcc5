"""GPU gather (e) vs the reference's gather fixtures (renderGBuffer + the
pipeline.hpp:161-207 stages) and vs the oracle on a 1080p property check.

Inputs are made identical first (the golden atlas and probe state are uploaded),
so each stage is compared on its own: integer stages (checkerboard downsample,
pixel selection, anchors, task count) exactly; floating stages in FP64 within
1e-9 relative where only the reference's arithmetic is involved, within 1e-6
where libm exp/pow enter (bilateral weights), and within the north-star 1e-3 for
Contact GI (its cosine directions carry sin/cos ulps into full traces).
"""
import os
import sys

import numpy as np
import pytest

from golden_util import GATHER_CASES, load_gather
from paper_2007_14394_b200 import api
from paper_2007_14394_b200.runtime import Device

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    d = Device(0, precision="f64")
    yield d
    d.close()


def rel(got, want, floor_frac=0.05):
    floor = floor_frac * max(float(np.mean(np.abs(want))), 1e-12)
    return np.abs(got - want) / np.maximum(np.abs(want), floor)


@pytest.mark.parametrize("name", GATHER_CASES)
def test_gather_matches_reference(dev, name):
    g = load_gather(name)
    src = g.src
    stage = api.ProbeStage(dev, g.scene, cfg=src.cfg(), res=src.res, spacing=src.spacing)
    for level in range(stage.levels):
        dev.upload_probes(level, g.data[f"gprobes_c{level}"])
        dev.upload_atlas(level, g.data[f"gatlas_c{level}"], which=0)
    cfg = stage.cfg
    # the G-buffer rendered on the device vs renderGBuffer
    dev.render_gbuffer(g.scene.camera, g.w, g.h, cfg)
    gb = dev.gbuffer()
    want = g.data["gbuffer"]
    sky = ~np.isfinite(want["depth"])
    assert np.array_equal(~np.isfinite(gb["depth"]), sky)
    geo = ~sky
    assert np.mean(gb["prim_index"][geo] == want["prim_index"][geo]) > 0.999
    assert np.allclose(gb["depth"][geo], want["depth"][geo], rtol=1e-9)
    # gather stages on the reference's own G-buffer
    dev.upload_gbuffer(g.w, g.h, want)
    dev.reset_history()
    for f, meta in enumerate(g.frames):
        n = dev.gather(f, cfg)
        assert n == meta["tasks"], (name, f)
        for k in ("half_src", "sel", "sparse_anchor", "sparse_valid"):
            assert np.array_equal(dev.gather_buffer(k), g.data[f"{k}_f{f}"]), (name, f, k)
        assert np.array_equal(dev.gather_buffer("half_depth"), g.data[f"half_depth_f{f}"])
        e = rel(dev.gather_buffer("sparse_irr"), g.data[f"sparse_irr_f{f}"])
        assert e.max() <= 1e-9, (name, f, "sparse_irr", e.max())
        e = rel(dev.gather_buffer("resolved"), g.data[f"resolved_f{f}"])
        assert e.max() <= 1e-6, (name, f, "resolved", e.max())
        e = rel(dev.gather_buffer("indirect"), g.data[f"indirect_f{f}"])
        assert np.mean(e > 1e-3) <= 1e-3 and e.max() <= 5e-2, (name, f, "indirect", e.max())


@pytest.mark.parametrize("name", GATHER_CASES)
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_compose_matches_reference(name, precision):
    """composeFrame (f1) on the reference's own G-buffer and indirect image: FP64
    bit-identical to the reference with identical shadow-trace statistics; FP32
    within the north-star 1e-3."""
    g = load_gather(name)
    src = g.src
    with Device(0, precision=precision) as d:
        stage = api.ProbeStage(d, g.scene, cfg=src.cfg(), res=src.res, spacing=src.spacing)
        d.upload_gbuffer(g.w, g.h, g.data["gbuffer"])
        for f, meta in enumerate(g.frames):
            d.upload_indirect(g.data[f"indirect_f{f}"])
            img, ms, st = d.compose(stage.cfg, stats=True)
            want = g.data[f"composed_f{f}"]
            if precision == "f64":
                assert np.array_equal(img, want), (name, f, float(np.max(np.abs(img - want))))
                ps = meta["compose_stats"]
                assert int(st["shadow_traces"]) == ps["shadow_traces"]
                assert int(st["sdf_queries"]) == ps["sdf_queries"]
            else:
                e = rel(img, want)
                assert np.mean(e > 1e-3) <= 1e-3 and e.max() <= 5e-2, (name, f, e.max())


def test_gather_1080p_properties(dev):
    """C3 at full size on the C2 scene: the G-buffer rendered on the device agrees with
    the oracle on a row sample; resolved irradiance is finite, >= 0, zero on sky."""
    from paper_2007_14394_b200 import scene_io

    scene = scene_io.read_sdfs(os.path.join(ROOT, "paper_2007_14394_b200", "data", "c2.sdfs"))
    stage = api.ProbeStage(dev, scene)
    for p in range(3):
        stage.run_pass(p)
    # G-buffer parity with the oracle at a size the CPU finishes quickly
    sw, sh = 160, 90
    dev.render_gbuffer(scene.camera, sw, sh, stage.cfg)
    small = dev.gbuffer()
    ogb, _ = oracle_py.Stage(scene).render_gbuffer(sw, sh)
    assert np.array_equal(np.isfinite(small["depth"]), np.isfinite(ogb["depth"]))
    geo = np.isfinite(ogb["depth"])
    assert np.mean(small["prim_index"][geo] == ogb["prim_index"][geo]) > 0.999
    w, h = 1920, 1080
    dev.render_gbuffer(scene.camera, w, h, stage.cfg)
    gb = dev.gbuffer()
    dev.reset_history()
    for f in range(2):
        dev.gather(f, stage.cfg)
        res = dev.gather_buffer("resolved").reshape(h * w, 3)
        ind = dev.gather_buffer("indirect").reshape(h * w, 3)
        assert np.all(np.isfinite(res)) and np.all(res >= 0) and np.all(np.isfinite(ind)) and np.all(ind >= 0)
        sky = ~np.isfinite(gb["depth"])
        assert np.all(res[sky] == 0) and np.all(ind[sky] == 0)
