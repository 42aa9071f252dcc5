"""C4: the large open scene — a ground plane (unbounded cluster) plus
50k primitives over 240 x 20 x 240 m, clustered by the library's linear-time
builder. Exactness vs the oracle on the full scene (queries on and off the
candidate grid, relocation of a sub-volume), and a small probe pass."""
import os
import sys

import numpy as np
import pytest

from paper_2007_14394_b200 import api, scenegen
from paper_2007_14394_b200.runtime import Device

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c4():
    return scenegen.with_fast_clusters(scenegen.c4_scene(50000), 8)


@pytest.mark.parametrize("margin", [None, ("0.6", "0")], ids=["default-grid", "tight-grid"])
def test_c4_queries_bit_exact(c4, margin, monkeypatch):
    if margin:  # a grid below the probe volume's top (the per-axis 0.6 margin)
        monkeypatch.setenv("SDFGI_GRID_MARGIN", margin[0])
        monkeypatch.setenv("SDFGI_GRID_MARGIN_MIN", margin[1])
    with Device(0, precision="f64") as dev:
        dev.upload_scene(c4)
        info = dev.accel_info()
        assert info["grid"]
        ora = oracle_py.Stage(c4)
        rng = np.random.default_rng(4)
        pts = np.concatenate([rng.uniform([-125, -2, -125], [125, 25, 125], size=(1500, 3)),
                              rng.uniform([-300, 30, -300], [300, 200, 300], size=(200, 3))])
        d_g, o_g = dev.query_points(pts)
        d_o, o_o = ora.query(pts)
        assert np.array_equal(d_g, d_o)
        assert np.array_equal(o_g, o_o)
        # the C4 probe volume reaches y = 60, above the geometry grid: setting the
        # cascade grows the grid over it (far cells end in truncated lists)
        dim0 = info["dim"]
        cs = c4.cascade
        api.makeCascade(dev, *cs.res, cs.spacing, 0, c4.camera.position)
        info = dev.accel_info()
        assert info["grid"]
        if margin:
            assert info["dim"] != dim0
        d_g, o_g = dev.query_points(pts)
        assert np.array_equal(d_g, d_o)
        assert np.array_equal(o_g, o_o)


def test_c4_relocation_and_pass_subvolume(c4):
    """A 24x8x24 sub-volume at the C4 spacing: bit-exact relocation vs the oracle and
    identical ray counts / probe states after one pass (every 16th probe)."""
    res = (24, 8, 24)
    with Device(0, precision="f64") as dev:
        stage = api.ProbeStage(dev, c4, res=res, n_rays=32)
        ora = oracle_py.Stage(c4, cfg=stage.cfg, res=res)
        stage.relocate_all()
        ora.relocate_all()
        g, o = dev.probes(0), ora.probes(0)
        for f in ("pos", "alive", "reject_history"):
            assert np.array_equal(g[f], o[f]), f
        n = res[0] * res[1] * res[2]
        refs = np.array([[0, i] for i in range(0, n, 16)], np.int32)
        r = api.updateProbes(dev, stage.cfg, 0, refs=refs)
        dev.swap()
        md, rays, upd, _ = ora.update(0, stride=16, threads=os.cpu_count() or 1)
        assert int(r["rays_traced"]) == rays and int(r["probes_updated"]) == upd
        ga, oa = dev.atlas(0), ora.atlas(0)
        floor = 0.05 * max(float(np.mean(np.abs(oa))), 1e-12)
        err = np.abs(ga.astype(np.float64) - oa) / np.maximum(np.abs(oa), floor)
        assert err.max() <= 1e-3, err.max()
