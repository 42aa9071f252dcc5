"""Known-answer tests of the device relocation (updateProbePositions) restating the
reference's own unit tests (test_probe_volume.cpp:26-112) through the
public API: the same single-box scenes, cascades and thresholds, in both modes
(relocation always runs in FP64)."""
import math

import numpy as np
import pytest

from paper_2007_14394_b200 import api, scene_io as sio
from paper_2007_14394_b200 import scene_file as sf
from paper_2007_14394_b200.runtime import Device

pytestmark = pytest.mark.gpu


def box_stage(dev, pos, half, res, cam):
    """boxScene (test_probe_volume.cpp:11-22) + makeCascade(res, spacing 1, level 0, cam)."""
    p = sf.Primitive(0, sio.BOX, sf.IDENTITY, tuple(map(float, pos)), tuple(map(float, half)), (0.5,) * 3, (0.0,) * 3,
                     0)
    cl = sf.buildClusters([p], 8, 10)
    camera = sio.Camera(np.array(cam, float), np.array([0, 0, -1.0]), np.array([1.0, 0, 0]), np.array([0, 1.0, 0]),
                        60.0)
    scene = sf.packScene([p], cl, np.zeros(0, sio.LIGHT_DTYPE), (0.0, 0.0, 0.0), camera,
                         sio.CascadeSpec(res, 1.0, 1), sio.default_cfg())
    return api.ProbeStage(dev, scene)


def set_history(dev, reject, last):
    pr = dev.probes(0)
    pr["reject_history"][:] = reject
    pr["last_update_frame"][:] = last
    dev.upload_probes(0, pr)


@pytest.fixture(scope="module")
def dev():
    d = Device(0, precision="f64")
    yield d
    d.close()


def test_probe_far_from_geometry_stays_at_its_grid_position(dev):
    box_stage(dev, (100, 0, 0), (1, 1, 1), (2, 2, 2), (0, 0, 0))
    set_history(dev, 0, 0)
    rep = api.updateProbePositions(dev, 0, 0.15, 0.3)
    assert int(rep["relocated"]) == 0 and int(rep["dead"]) == 0
    pr = dev.probes(0)
    assert np.all(np.linalg.norm(pr["pos"] - pr["resting"], axis=1) < 1e-12)
    assert pr["reject_history"][0] == 0


def test_probe_just_inside_a_wall_is_pushed_out_past_the_clearance_threshold(dev):
    th1 = 0.1
    box_stage(dev, (-4.49, 0.5, 0.5), (5, 5, 5), (2, 2, 2), (1, 1, 1))
    resting = dev.probes(0)["resting"][0]
    d0, _ = api.querySceneSdf(dev, resting[None, :])
    assert abs(d0[0] - (-0.01)) <= 1e-9
    rep = api.updateProbePositions(dev, 0, th1, 0.3)
    probe = dev.probes(0)[0]
    assert probe["alive"] == 1 and int(rep["relocated"]) >= 1
    d1, _ = api.querySceneSdf(dev, probe["pos"][None, :])
    assert d1[0] >= th1
    # brute-force oracle along the gradient line (sceneGradient, h = 1e-3)
    h = 1e-3
    offs = np.array([[h, 0, 0], [-h, 0, 0], [0, h, 0], [0, -h, 0], [0, 0, h], [0, 0, -h]])
    dd, _ = api.querySceneSdf(dev, resting[None, :] + offs)
    g = np.array([dd[0] - dd[1], dd[2] - dd[3], dd[4] - dd[5]])
    g /= np.linalg.norm(g)
    ts = np.arange(0, 0.5, 1e-4)
    dl, _ = api.querySceneSdf(dev, resting[None, :] + ts[:, None] * g[None, :])
    oracle = ts[np.argmax(dl >= th1)]
    moved = np.linalg.norm(probe["pos"] - resting)
    assert moved <= oracle + 0.5 * th1 and moved <= 0.5


def test_relocation_is_idempotent_in_a_static_scene(dev):
    box_stage(dev, (0.2, 0, 0), (1, 1, 1), (3, 3, 3), (0, 0, 0))
    api.updateProbePositions(dev, 0, 0.15, 0.3)
    set_history(dev, 0, 0)
    first = dev.probes(0)["pos"].copy()
    rep = api.updateProbePositions(dev, 0, 0.15, 0.3)
    assert int(rep["rejected"]) == 0
    pr = dev.probes(0)
    assert np.all(np.linalg.norm(pr["pos"] - first, axis=1) < 1e-12)
    assert np.all(pr["reject_history"] == 0)


def test_probe_trapped_deep_inside_geometry_is_marked_dead(dev):
    box_stage(dev, (0.5, 0.5, 0.5), (3, 3, 3), (2, 2, 2), (1, 1, 1))
    rep = api.updateProbePositions(dev, 0, 0.15, 0.3)
    assert int(rep["dead"]) == 8 and np.all(dev.probes(0)["alive"] == 0)


def test_large_relocation_rejects_history_and_is_reported(dev):
    box_stage(dev, (100, 0, 0), (1, 1, 1), (2, 2, 2), (1, 1, 1))
    api.updateProbePositions(dev, 0, 0.15, 0.3)
    set_history(dev, 0, 1)
    before = dev.probes(0)
    # the wall arrives next frame: same cascade, new scene (surface at x = 0.6)
    wall = box_stage(dev, (-4.4, 0.5, 0.5), (5, 5, 5), (2, 2, 2), (1, 1, 1))
    dev.upload_probes(0, before)
    rep = api.updateProbePositions(dev, 0, 0.3, 0.3)
    assert int(rep["rejected"]) > 0 and np.any(dev.probes(0)["reject_history"] == 1)
    del wall
