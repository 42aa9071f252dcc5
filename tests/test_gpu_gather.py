"""GPU gather (e) vs the reference's gather fixtures (renderGBuffer + the
pipeline.hpp:161-207 stages) and vs the oracle on a 1080p property check.

Inputs are made identical first (the golden atlas and probe state are uploaded),
so each stage is compared on its own: integer stages (checkerboard downsample,
pixel selection, anchors, task count) exactly; floating stages in FP64 within
1e-9 relative where only the reference's arithmetic is involved, within 1e-6
where libm exp/pow enter (bilateral weights), and within the north-star 1e-3 on
every channel for Contact GI (its cosine directions are bit-identical: the
sin/cos come from the host's libm, host_trig.h).
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
    assert np.array_equal(gb["prim_index"], want["prim_index"])
    assert np.array_equal(gb["depth"][geo], want["depth"][geo])
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
        assert e.max() <= 1e-3, (name, f, "indirect", e.max())


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


def test_gather_1080p_matches_oracle(dev, oracle_c2):
    """C3 (BASELINE configs[2]) at full size against the oracle: the 1920x1080 gather
    on the C2 scene and volume after its 3 bounces (the oracle's probe state and
    atlas uploaded, so the gather is compared on identical inputs). The device
    G-buffer equals renderGBuffer's bit for bit; two frames (the second with
    history): integer stages exact, sparse irradiance 1e-9, resolved 1e-6 (libm
    exp/pow in the bilateral weights), indirect (Contact GI) within 1e-3 on every
    channel."""
    scene, ora = oracle_c2["scene"], oracle_c2["stage"]
    last = oracle_c2["passes"][-1]
    stage = api.ProbeStage(dev, scene)
    dev.upload_probes(0, last["probes"])
    dev.upload_atlas(0, last["atlas"], which=0)
    cfg = stage.cfg
    w, h = 1920, 1080
    ogb, _ = ora.render_gbuffer(w, h)
    dev.render_gbuffer(scene.camera, w, h, cfg)
    gb = dev.gbuffer()
    assert np.array_equal(gb["prim_index"], ogb["prim_index"])
    geo = np.isfinite(ogb["depth"])
    assert np.array_equal(np.isfinite(gb["depth"]), geo)
    assert np.array_equal(gb["depth"][geo], ogb["depth"][geo])
    assert np.array_equal(gb["normal"][geo], ogb["normal"][geo])
    dev.reset_history()
    hist = None
    for f in range(2):
        want = ora.gather_frame(ogb, w, h, f, hist)
        n = dev.gather(f, cfg)
        assert n == want["tasks"], f
        for k in ("half_src", "sel", "sparse_anchor", "sparse_valid", "half_depth"):
            assert np.array_equal(dev.gather_buffer(k), want[k]), (f, k)
        e = rel(dev.gather_buffer("sparse_irr"), want["sparse_irr"])
        assert e.max() <= 1e-9, (f, "sparse_irr", e.max())
        e = rel(dev.gather_buffer("resolved"), want["resolved"])
        assert e.max() <= 1e-6, (f, "resolved", e.max())
        ind = dev.gather_buffer("indirect")
        e = rel(ind, want["indirect"])
        print(f"C3 frame {f}: indirect max rel err {e.max():.3e}, bit-identical {np.mean(ind == want['indirect']):.6f}")
        assert e.max() <= 1e-3, (f, "indirect", e.max())
        hist = (want["resolved"], ogb["depth"].copy())
