"""Known-answer tests of the device sphere tracer and query seeding, restating the
reference's test_trace.cpp:82-164 through the public API: probe rays
(sdfgi_probes_trace_debug) against analytic intersections, and the seeded query
contract along random marches (sdfgi_query_points with initD = 2 * lastD)."""
import math

import numpy as np
import pytest

from paper_2007_14394_b200 import api, scene_io as sio
from paper_2007_14394_b200 import scene_file as sf
from paper_2007_14394_b200.runtime import Device

pytestmark = pytest.mark.gpu
EPS = 1e-3  # RenderConfig::surfaceEpsilon


def stage_of(dev, prims, res, cam, n_rays=64):
    cl = sf.buildClusters(prims, 8, 10)
    camera = sio.Camera(np.array(cam, float), np.array([0, 0, -1.0]), np.array([1.0, 0, 0]), np.array([0, 1.0, 0]),
                        60.0)
    scene = sf.packScene(prims, cl, np.zeros(0, sio.LIGHT_DTYPE), (0.0, 0.0, 0.0), camera,
                         sio.CascadeSpec(res, 1.0, 1), sio.default_cfg(n_rays_full=n_rays))
    return api.ProbeStage(dev, scene)


def prim(pid, kind, size, pos, rot=sf.IDENTITY):
    return sf.Primitive(pid, kind, rot, tuple(map(float, pos)), tuple(map(float, size)), (0.5,) * 3, (0.0,) * 3, 0)


def ray_sphere(o, d, c, r):
    oc = o - c
    b = np.dot(oc, d)
    disc = b * b - (np.dot(oc, oc) - r * r)
    if disc < 0:
        return None
    t = -b - math.sqrt(disc)
    return t if t > 0 else None


def ray_box(o, d, c, h):
    with np.errstate(divide="ignore"):
        inv = 1.0 / d
    t0, t1 = (c - h - o) * inv, (c + h - o) * inv
    tn, tf = np.max(np.minimum(t0, t1)), np.min(np.maximum(t0, t1))
    return tn if tf >= tn and tn > 0 else None


def box_normal(p, c, h):
    q = (p - c) / h
    n = np.zeros(3)
    a = int(np.argmax(np.abs(q)))
    n[a] = 1.0 if q[a] > 0 else -1.0
    return n


CASES = {
    "sphere": ([prim(0, sio.SPHERE, (1.3, 0, 0), (0.5, -0.3, 0.2))], (0.5, -0.3, 0.2),
               lambda o, d: ray_sphere(o, d, np.array([0.5, -0.3, 0.2]), 1.3),
               lambda p: (p - np.array([0.5, -0.3, 0.2])) / np.linalg.norm(p - np.array([0.5, -0.3, 0.2]))),
    "box": ([prim(1, sio.BOX, (1, 0.8, 1.4), (0, 0.5, -0.5))], (0, 0.5, -0.5),
            lambda o, d: ray_box(o, d, np.array([0, 0.5, -0.5]), np.array([1, 0.8, 1.4])),
            lambda p: box_normal(p, np.array([0, 0.5, -0.5]), np.array([1, 0.8, 1.4]))),
    "plane": ([prim(2, sio.PLANE, (1, 1, 1), (0, -1, 0), sf.fromZTo((0.0, 1.0, 0.0)))], (0, 0.5, 0),
              lambda o, d: ((-1.0 - o[1]) / d[1]) if d[1] < 0 else None,
              lambda p: np.array([0.0, 1.0, 0.0])),
}


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("name", list(CASES))
def test_probe_rays_match_analytic_intersections(name, precision):
    prims, target, oracle, normal_at = CASES[name]
    with Device(0, precision=precision) as dev:
        stage = stage_of(dev, prims, (5, 5, 5), target)
        stage.relocate_all()
        pr = dev.probes(0)
        refs = np.array([[0, i] for i in range(len(pr)) if pr["alive"][i]], np.int32)
        recs = dev.trace_debug(0, stage.cfg, refs)
        n = len(recs) // len(refs)
        tested = 0
        for k, (_, i) in enumerate(refs):
            o = pr["pos"][i]
            for r in recs[k * n:(k + 1) * n]:
                d = r["dir"]
                t = oracle(o, d)
                if t is None or t > 99:
                    continue
                if abs(np.dot(normal_at(o + d * t), d)) < 0.3:  # near-tangent incidence
                    continue
                assert r["converged"] == 1, (name, i)
                assert abs(r["t"] - t) <= 2 * EPS, (name, i, r["t"], t)
                tested += 1
        assert tested >= 1000, tested


def test_seeding_never_changes_a_step():
    rng = np.random.default_rng(23)
    prims = [prim(0, sio.SPHERE, (1, 0, 0), (2, 0, 0)),
             prim(1, sio.BOX, (0.8, 1.5, 0.6), (-2, 0.5, 1), sf.fromAxisAngle((0.0, 1.0, 0.0), 0.6)),
             prim(2, sio.CAPSULE, (0.4, 1.0, 0), (0, -2, -1))]
    with Device(0, precision="f64") as dev:
        stage_of(dev, prims, (2, 2, 2), (0, 0, 0))
        o = rng.uniform(-6, 6, size=(4000, 3))
        d0, _ = api.querySceneSdf(dev, o)
        o = o[d0 > 0][:1000]
        assert len(o) == 1000
        d = rng.normal(size=(1000, 3))
        d /= np.linalg.norm(d, axis=1)[:, None]
        t = np.zeros(1000)
        last = np.full(1000, np.inf)
        live = np.ones(1000, bool)
        for _ in range(128):
            p = o + d * t[:, None]
            un, _ = api.querySceneSdf(dev, p)
            assert np.all(un[live] >= 0.0)  # never inside geometry
            init = np.where(np.isinf(last), np.inf, 2 * last)
            se, _ = api.querySceneSdf(dev, p, init)
            chk = live & ~np.isinf(last) & (un < 2 * last)
            assert np.array_equal(se[chk], un[chk])
            live &= ~(un < EPS)
            t = np.where(live, t + un, t)
            last = np.where(live, un, last)
            live &= t <= 50
            if not live.any():
                break
