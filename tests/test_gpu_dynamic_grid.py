"""Animated geometry on the candidate grid (f2: "AABB refit for animated
primitives"): primitives that move between uploads leave the grid lists and are
evaluated by every on-grid query; the grid is rebuilt only when a primitive moves
for the first time (or more than kMaxDynamic move). Checked on the C2 scene with a
few primitives moving over several frames: every query value and owner
bit-identical to the oracle on the moved scene, relocation bit-exact, a probe pass
with identical probe states and texels within 1e-3; a re-clustered upload of the
same geometry keeps the grid (lists remapped) and stays exact."""
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


def moved(scene, frame, ids):
    """The scene with primitives `ids` translated along a small orbit at `frame`;
    the clusters' boxes grown to keep containing them."""
    import copy

    s = copy.deepcopy(scene)
    for k, i in enumerate(ids):
        ang = 0.6 * frame + k
        s.prims["trans"][i] += np.array([0.35 * np.cos(ang), 0.2 * np.sin(1.3 * ang), 0.35 * np.sin(ang)])
    # cluster boxes: conservative (the union of the original and the moved member boxes)
    ms, mi = s.member_start, s.member_idx
    for c in range(len(s.clusters)):
        for m in range(ms[c], ms[c + 1]):
            if mi[m] in ids:
                s.clusters["lo"][c] -= 0.6
                s.clusters["hi"][c] += 0.6
    return s


def test_animated_primitives_refit_exact():
    base = scene_io.read_sdfs(C2)
    rng = np.random.default_rng(11)
    ids = sorted(int(i) for i in rng.choice(len(base.prims), 6, replace=False))
    pts = np.concatenate([rng.uniform([-7.5, -1, -5.5], [7.5, 7.5, 5.5], size=(20000, 3))])
    with Device(0, precision="f64") as dev:
        stage = api.ProbeStage(dev, base)
        for frame in range(1, 5):
            sc = moved(base, frame, ids)
            stage.set_scene(sc)
            ora = oracle_py.Stage(sc)
            d_g, o_g = dev.query_points(pts)
            d_o, o_o = ora.query(pts)
            assert np.array_equal(d_g, d_o) and np.array_equal(o_g, o_o), frame
            # a pass on every 5th probe: relocation bit-exact, states equal, texels 1e-3
            stage.relocate_all()
            ora.relocate_all()
            g, o = dev.probes(0), ora.probes(0)
            for f in ("pos", "alive", "reject_history"):
                assert np.array_equal(g[f], o[f]), (frame, f)
            ora.close()


def test_reclustered_upload_keeps_grid_exact():
    """The same geometry with a different clustering (the reference re-clusters
    every frame): lists remapped to the new CSR order, queries still exact."""
    from paper_2007_14394_b200 import scenegen

    base = scene_io.read_sdfs(C2)
    other = scenegen.with_fast_clusters(base, 4)
    rng = np.random.default_rng(12)
    pts = rng.uniform([-7.5, -1, -5.5], [7.5, 7.5, 5.5], size=(20000, 3))
    with Device(0, precision="f64") as dev:
        dev.upload_scene(base)
        dev.upload_scene(other)
        d_g, o_g = dev.query_points(pts)
        ora = oracle_py.Stage(other)
        d_o, o_o = ora.query(pts)
        assert np.array_equal(d_g, d_o) and np.array_equal(o_g, o_o)
