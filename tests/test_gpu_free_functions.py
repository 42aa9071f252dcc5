"""The reference's free functions through the batched C-ABI entry points
(sdfgi_trace_rays, sdfgi_soft_shadow, sdfgi_shade_hits, sdfgi_convolve_irradiance,
sdfgi_interpolation_stencil; api.py mirrors). Known answers restated from the
reference's tests: sphere trace vs analytic intersection (test_trace.cpp:82-135),
soft shadow clear/blocked (:166-230), the E = 4 pi / N estimator (test_probe_update.
cpp:74-102), shadeHit emission (:104-144), stencil partition of unity and
trilinear weights (test_probe_volume.cpp:182-205). Bit parity of the same entry
points against the reference itself: tests/test_dropin.py::test_dropin_free_functions."""
import math

import numpy as np
import pytest

from paper_2007_14394_b200 import api, runtime, scene_io as sio
from paper_2007_14394_b200.runtime import Device
from test_gpu_trace_kats import EPS, prim, ray_sphere, stage_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    d = Device(0, precision="f64")
    yield d
    d.close()


def sphere_stage(dev):
    return stage_of(dev, [prim(0, sio.SPHERE, (1.3, 0, 0), (0.5, -0.3, 0.2))], (4, 4, 4), (0.0, 0.0, 0.0))


def test_sphere_trace_batch_matches_analytic(dev):
    sphere_stage(dev)
    rng = np.random.default_rng(1)
    o = rng.uniform(-6, 6, (2000, 3))
    o = o[np.linalg.norm(o - [0.5, -0.3, 0.2], axis=1) > 1.5]
    d = rng.normal(size=(len(o), 3))
    half = len(o) // 2  # half of the rays aimed near the sphere, half random
    d[:half] = np.array([0.5, -0.3, 0.2]) + rng.uniform(-1.5, 1.5, (half, 3)) - o[:half]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    h = api.sphereTrace(dev, o, d, 100.0, EPS, 128)
    for i in range(len(o)):
        t = ray_sphere(o[i], d[i], np.array([0.5, -0.3, 0.2]), 1.3)
        if t is None:  # a near miss may still converge within eps of the surface (d < eps)
            if h["converged"][i]:
                assert abs(np.linalg.norm(h["pos"][i] - [0.5, -0.3, 0.2]) - 1.3) <= EPS
            else:
                assert h["miss"][i] in (1, 2)
        elif h["converged"][i]:
            # on the surface to the polish tolerance; t within 2 eps unless grazing
            c = np.array([0.5, -0.3, 0.2])
            assert abs(np.linalg.norm(h["pos"][i] - c) - 1.3) <= EPS and h["prim_index"][i] == 0
            n = (h["pos"][i] - c) / np.linalg.norm(h["pos"][i] - c)
            if -np.dot(n, d[i]) > 0.2:
                assert abs(h["t"][i] - t) <= 2 * EPS
            assert np.allclose(h["normal"][i], n, atol=1e-5)
    assert np.mean(h["converged"]) > 0.2


def test_soft_shadow_batch_clear_and_blocked(dev):
    sphere_stage(dev)
    c = np.array([0.5, -0.3, 0.2])
    o = np.array([[5.0, 5.0, 5.0], c + [3.0, 0, 0]])
    d = np.array([[0.0, 1.0, 0.0], [-1.0, 0.0, 0.0]])
    v = api.softShadowTrace(dev, o, d, 0.01, 10.0, 8.0)
    assert v[0] == 1.0  # away from everything
    assert v[1] == 0.0  # straight through the sphere


def test_convolve_estimator_known_answers(dev):
    """E = 4 pi / N sum max(0, D.d) L: one sample along D with L = 1 gives 4 pi / 1;
    a sample behind D contributes nothing; empty input gives 0."""
    D = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]])
    e = api.convolveIrradiance(dev, [[0.0, 0.0, 1.0]], [[1.0, 2.0, 3.0]], D)
    assert np.allclose(e[0], 4 * math.pi * np.array([1.0, 2.0, 3.0]), rtol=1e-15)
    assert np.all(e[1] == 0)
    rng = np.random.default_rng(3)
    sd = rng.normal(size=(257, 3))
    sd /= np.linalg.norm(sd, axis=1, keepdims=True)
    sr = rng.uniform(size=(257, 3))
    td = rng.normal(size=(64, 3))
    td /= np.linalg.norm(td, axis=1, keepdims=True)
    got = api.convolveIrradiance(dev, sd, sr, td)
    for t in range(64):  # the reference's summation order, in Python floats
        acc = [0.0, 0.0, 0.0]
        for i in range(257):
            w = td[t, 0] * sd[i, 0] + td[t, 1] * sd[i, 1] + td[t, 2] * sd[i, 2]
            if w > 0:
                acc = [acc[k] + sr[i, k] * w for k in range(3)]
        want = [a * (4.0 * math.pi / 257) for a in acc]
        assert np.array_equal(got[t], np.array(want))


def test_shade_hit_emission_and_sky(dev):
    """shadeHit: no lights, no field -> emission; no owner -> the sky."""
    from paper_2007_14394_b200 import scene_file as sf

    p = sf.Primitive(0, sio.SPHERE, sf.IDENTITY, (0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.5,) * 3, (5.0, 5.0, 5.0), 0)
    stage = stage_of(dev, [p], (4, 4, 4), (0.0, 0.0, 0.0))
    h = np.zeros(2, runtime.HIT_DTYPE)
    h["converged"] = 1
    h["pos"][0] = [1.0, 0, 0]
    h["normal"][0] = [1.0, 0, 0]
    h["prim_index"] = [0, -1]
    rad = api.shadeHit(dev, h, 0.0, stage.cfg)
    assert np.array_equal(rad[0], [5.0, 5.0, 5.0])
    assert np.array_equal(rad[1], [0.0, 0.0, 0.0])  # the scene's sky


def test_interpolation_stencil_partition_and_trilinear(dev):
    """Undisplaced probes (no relocation): trilinear weights of the cell, summing to 1;
    outside every cascade: sky fallback."""
    stage = stage_of(dev, [prim(0, sio.SPHERE, (0.1, 0, 0), (50.0, 50.0, 50.0))], (4, 4, 4), (0.0, 0.0, 0.0))
    res, sp, origin = dev.levels[0]
    rng = np.random.default_rng(5)
    pts = origin + rng.uniform(0.01, 2.99, (500, 3)) * sp
    st = api.interpolationStencil(dev, pts)
    assert np.all(st["count"] == 8) and np.all(st["sky_fallback"] == 0) and np.all(st["used_mvc"] == 0)
    assert np.allclose(st["weight"].sum(axis=1), 1.0, atol=1e-12)
    f = (pts - origin) / sp
    cell = np.floor(f).astype(int)
    t = f - cell
    for k in range(8):
        wx = np.where(k & 1, t[:, 0], 1 - t[:, 0])
        wy = np.where((k >> 1) & 1, t[:, 1], 1 - t[:, 1])
        wz = np.where((k >> 2) & 1, t[:, 2], 1 - t[:, 2])
        assert np.allclose(st["weight"][:, k], wx * wy * wz, atol=1e-12)
        idx = (cell[:, 0] + (k & 1)) + res[0] * ((cell[:, 1] + ((k >> 1) & 1)) + res[1] * (cell[:, 2] + ((k >> 2) & 1)))
        assert np.array_equal(st["index"][:, k], idx)
    far = api.interpolationStencil(dev, [[1e3, 1e3, 1e3]])
    assert far["sky_fallback"][0] == 1 and far["count"][0] == 0 and far["cross_cascade"][0] == 1
