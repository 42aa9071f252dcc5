"""Known-answer tests of the device probe stage, restating the reference's own unit
tests (test_probe_update.cpp:146-294) through the public API: the
same hollow-room scenes (six emissive slabs, clusters from the reference's
buildClusters), the same cascades, configs and tolerances."""
import math

import numpy as np
import pytest

from paper_2007_14394_b200 import api, scene_io as sio
from paper_2007_14394_b200 import scene_file as sf
from paper_2007_14394_b200.runtime import Device

pytestmark = pytest.mark.gpu


def room_scene(half, thick, emission, albedo):
    """roomScene, test_probe_update.cpp:21-37: interior [-half, half]^3 in six slabs."""
    c, w = half + thick / 2, half + thick
    boxes = [((c, 0, 0), (thick / 2, w, w)), ((-c, 0, 0), (thick / 2, w, w)), ((0, c, 0), (w, thick / 2, w)),
             ((0, -c, 0), (w, thick / 2, w)), ((0, 0, c), (w, w, thick / 2)), ((0, 0, -c), (w, w, thick / 2))]
    prims = [sf.Primitive(i, sio.BOX, sf.IDENTITY, tuple(map(float, p)), tuple(map(float, e)),
                          tuple(map(float, albedo)), tuple(map(float, emission)), 0) for i, (p, e) in enumerate(boxes)]
    return prims, sf.buildClusters(prims, 8, 100)


def make(dev, prims, clusters, res, origin_cam, cfg, sky=(0.0, 0.0, 0.0)):
    cam = sio.Camera(np.array(origin_cam, float), np.array([0, 0, -1.0]), np.array([1.0, 0, 0]),
                     np.array([0, 1.0, 0]), 60.0)
    scene = sf.packScene(prims, clusters, np.zeros(0, sio.LIGHT_DTYPE), sky, cam, sio.CascadeSpec(res, 1.0, 1), cfg)
    return api.ProbeStage(dev, scene)


def lum(t):
    return 0.2126 * t[..., 0] + 0.7152 * t[..., 1] + 0.0722 * t[..., 2]  # vec.hpp:72


def interior(atlas, probe):
    return atlas[probe, 1:-1, 1:-1, :].astype(np.float64)


@pytest.fixture(params=["f64", "f32"])
def dev(request):
    d = Device(0, precision=request.param)
    yield d
    d.close()


def test_furnace_converges_to_pi_in_one_rejected_update(dev):
    prims, cl = room_scene(2, 0.4, (1, 1, 1), (0, 0, 0))
    stage = make(dev, prims, cl, (2, 2, 2), (0.5, 0.5, 0.5), sio.default_cfg(n_rays_full=512, bounce_coeff=0))
    stage.relocate_all()
    assert dev.probes(0)["reject_history"][0] == 1
    r = api.updateProbes(dev, stage.cfg, 0, refs=np.array([[0, 0]], np.int32))
    assert int(r["rays_traced"]) == 1024
    dev.swap()
    assert np.allclose(interior(dev.atlas(0, 0), 0), math.pi, rtol=0.05)


def test_pure_sky_scene_converges_to_sky_irradiance(dev):
    sky = (0.5, 0.25, 1.0)
    stage = make(dev, [], [], (2, 2, 2), (0, 0, 0), sio.default_cfg(bounce_coeff=0), sky)
    for f in range(3):
        stage.run_pass(f)
    t = dev.atlas(0, 0)[0, 1 + 3, 1 + 3]
    assert np.allclose(t, math.pi * np.array(sky), rtol=0.05)


def test_history_rejection_replaces_texels_with_the_single_frame_estimate(dev):
    prims, cl = room_scene(2, 0.4, (1, 1, 1), (0, 0, 0))
    out = []
    for garbage in (0.0, 123.0):
        stage = make(dev, prims, cl, (2, 2, 2), (0.5, 0.5, 0.5), sio.default_cfg(n_rays_full=64, bounce_coeff=0))
        stage.relocate_all()
        t = dev.oct_res + 2
        dev.upload_atlas(0, np.full((8, t, t, 3), garbage, np.float32), which=0)
        pr = dev.probes(0)
        pr["reject_history"][0] = 1
        dev.upload_probes(0, pr)
        api.updateProbes(dev, stage.cfg, 7, refs=np.array([[0, 0]], np.int32))
        dev.swap()
        out.append(dev.atlas(0, 0)[0].copy())  # prior texel contents must not matter
    assert np.array_equal(out[0], out[1])


def test_static_furnace_approaches_its_fixed_point_at_ratio_0_9(dev):
    prims, cl = room_scene(2, 0.4, (1, 1, 1), (0, 0, 0))
    cfg = sio.default_cfg(n_rays_full=144, bounce_coeff=0, hysteresis=0.9)
    stage = make(dev, prims, cl, (2, 2, 2), (0.5, 0.5, 0.5), cfg)
    stage.relocate_all()
    lums = []
    for f in range(52):
        pr = dev.probes(0)
        pr["reject_history"][:] = 0  # the plain blending path from frame 0
        dev.upload_probes(0, pr)
        api.updateProbes(dev, stage.cfg, f)
        dev.swap()
        lums.append(float(np.mean(lum(interior(dev.atlas(0, 0), 0)))))
    k = np.arange(1, 30)
    delta = np.array([lums[i] - lums[i - 1] for i in k])
    assert np.all(delta > 0)
    slope = np.polyfit(k, np.log(delta), 1)[0]
    assert abs(math.exp(slope) - 0.9) <= 0.02


def test_multi_bounce_feedback_converges_to_the_geometric_series(dev):
    prims, cl = room_scene(2.0, 0.4, (1, 1, 1), (0.5, 0.5, 0.5))
    cfg = sio.default_cfg(n_rays_full=96, bounce_coeff=1.0, hysteresis=0.8)
    stage = make(dev, prims, cl, (6, 6, 6), (0, 0, 0), cfg)
    for f in range(90):
        stage.run_pass(f)
    expected = math.pi / (1.0 - 0.5)
    atlas = dev.atlas(0, 0)
    center = 2 + 6 * (2 + 6 * 2)
    assert abs(float(np.mean(lum(interior(atlas, center)))) - expected) <= 0.10 * expected
    assert float(np.max(interior(atlas, slice(None)))) <= expected * 1.1


def test_texels_never_go_negative(dev):
    prims, cl = room_scene(2, 0.3, (0.2, 1.5, 0.7), (0.6, 0.3, 0.8))
    stage = make(dev, prims, cl, (3, 3, 3), (0, 0, 0), sio.default_cfg(n_rays_full=32))
    for f in range(10):
        stage.run_pass(f)
    assert np.all(dev.atlas(0, 0) >= 0)


def test_probe_updates_are_deterministic(dev):
    prims, cl = room_scene(2, 0.4, (1, 0.5, 0.25), (0.4, 0.4, 0.4))
    out = []
    for _ in range(2):
        stage = make(dev, prims, cl, (3, 3, 3), (0, 0, 0), sio.default_cfg(n_rays_full=48))
        for f in range(4):
            stage.run_pass(f)
        out.append(dev.atlas(0, 0))
    assert np.array_equal(out[0], out[1])
