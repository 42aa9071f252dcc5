"""Deterministic synthetic scenes for the BASELINE configs.

C2 ("Sponza-scale"): the 7 shell boxes of the sponza-lite atrium (floor, four
walls, two aisle ceilings) plus 1,993 random primitives drawn with the
reference's own counter-based RNG (splitmix64 ``Rng``, rng.hpp:22-48, seed 1):
kinds uniform over {sphere, box, cylinder, capsule}, size ~ U(0.05, 0.25),
positions uniform over x in [-6.5, 6.5], y in [0, 5.8], z in [-4.5, 4.5], 30%
rotated about a random axis, albedo U(0.2, 0.8)^3, 2% emissive U(0, 2).
Lights and sky as sponza-lite (a directional sun and a point light). Camera at
(0, 3, 0) looking at (-4, 1.2, -0.6), fov 72, so ``makeCascade`` centres the
32x16x32 volume (spacing 0.45) on the atrium: origin (-6.975, -0.225, -6.975).

C4 ("large open"): a ground plane (unbounded cluster) plus N primitives over
x, z in [-120, 120], y in [0, 20], sizes U(0.2, 2.0), a sun and the
open-field sky; 128x32x128 probes at spacing 1.875.

Clusters are not built here: C2's were built once by the reference's
``buildClusters`` (scene.hpp:110-178, via oracle/ref_driver.cpp ``recluster``)
and committed in data/c2.sdfs; large scenes use the library's linear-time
builder (``with_fast_clusters`` -> ``sdfgi_build_clusters``).
"""
from __future__ import annotations

import math

import numpy as np

from . import scene_io as sio

M64 = (1 << 64) - 1


def _hash(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E9B5) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


class Rng:
    """rng.hpp:22-48 (splitmix64 stream keyed by a u64)."""

    def __init__(self, key):
        self.s = _hash(key & M64)

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E9B5) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def uniform(self, lo=0.0, hi=1.0):
        u = (self.next() >> 11) * (1.0 / (1 << 53))
        return lo + (hi - lo) * u


def axis_angle(axis, radians):
    """Mat3::fromAxisAngle, vec.hpp:80-94 (row-major)."""
    a = np.asarray(axis, float)
    a = a / math.sqrt(float(a @ a))
    c, s = math.cos(radians), math.sin(radians)
    t = 1 - c
    x, y, z = a
    return np.array(
        [t * x * x + c, t * x * y - s * z, t * x * z + s * y,
         t * x * y + s * z, t * y * y + c, t * y * z - s * x,
         t * x * z - s * y, t * y * z + s * x, t * z * z + c]
    )


def _prim(pid, kind, pos, size, rot=None, albedo=(0.5, 0.5, 0.5), emission=(0, 0, 0)):
    p = np.zeros(1, sio.PRIM_DTYPE)
    p["id"] = pid
    p["kind"] = kind
    p["rot"] = np.eye(3).reshape(9) if rot is None else rot
    p["trans"] = pos
    p["size"] = size
    p["albedo"] = albedo
    p["emission"] = emission
    return p


def _random_prims(rng: Rng, n, first_id, box_lo, box_hi, rmin, rmax):
    out = []
    for i in range(n):
        kind = [sio.SPHERE, sio.BOX, sio.CYLINDER, sio.CAPSULE][int(rng.uniform() * 4) % 4]
        pos = tuple(rng.uniform(box_lo[k], box_hi[k]) for k in range(3))
        r = rng.uniform(rmin, rmax)
        if kind == sio.SPHERE:
            size = (r, 0.0, 0.0)
        elif kind == sio.BOX:
            size = (r, rng.uniform(rmin, rmax), rng.uniform(rmin, rmax))
        else:
            size = (r, rng.uniform(rmin, 2 * rmax), 0.0)
        rot = None
        if rng.uniform() < 0.3:
            axis = (rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1))
            if sum(a * a for a in axis) < 1e-6:
                axis = (0.0, 1.0, 0.0)
            rot = axis_angle(axis, rng.uniform(0, 2 * math.pi))
        albedo = tuple(rng.uniform(0.2, 0.8) for _ in range(3))
        emission = (0.0, 0.0, 0.0)
        if rng.uniform() < 0.02:
            emission = tuple(rng.uniform(0.0, 2.0) for _ in range(3))
        out.append(_prim(first_id + i, kind, pos, size, rot, albedo, emission))
    return out


def _camera(pos, look_at, fov):
    """Camera::lookAt, camera.hpp:15-26."""
    pos = np.asarray(pos, float)
    f = np.asarray(look_at, float) - pos
    f = f / math.sqrt(float(f @ f))
    r = np.cross(f, [0.0, 1.0, 0.0])
    r = r / math.sqrt(float(r @ r))
    u = np.cross(r, f)
    return sio.Camera(pos, f, r, u, float(fov))


def c2_scene(n_random=1993, seed=1) -> sio.Scene:
    """SURVEY §8d C2 (unclustered; see data/c2.sdfs for the clustered file)."""
    shell = [
        ((0, -0.2, 0), (7, 0.2, 5), (0.62, 0.58, 0.54)),
        ((0, 3, -4.7), (7, 3.4, 0.2), (0.66, 0.62, 0.58)),
        ((0, 3, 4.7), (7, 3.4, 0.2), (0.66, 0.62, 0.58)),
        ((-6.7, 3, 0), (0.2, 3.4, 5), (0.66, 0.62, 0.58)),
        ((6.7, 3, 0), (0.2, 3.4, 5), (0.66, 0.62, 0.58)),
        ((0, 6.1, -3.4), (7, 0.15, 1.4), (0.6, 0.6, 0.6)),
        ((0, 6.1, 3.4), (7, 0.15, 1.4), (0.6, 0.6, 0.6)),
    ]
    prims = [_prim(i, sio.BOX, p, s, None, a) for i, (p, s, a) in enumerate(shell)]
    prims += _random_prims(Rng(seed), n_random, 100, (-6.5, 0.0, -4.5), (6.5, 5.8, 4.5), 0.05, 0.25)
    lights = np.zeros(2, sio.LIGHT_DTYPE)
    lights[0]["kind"] = sio.LIGHT_DIRECTIONAL
    d = np.array([0.25, -1.0, 0.15])
    lights[0]["direction"] = d / math.sqrt(float(d @ d))
    lights[0]["intensity"] = (2.2, 2.1, 1.9)
    lights[1]["kind"] = sio.LIGHT_POINT
    lights[1]["position"] = (0, 4.5, 0)
    lights[1]["intensity"] = (6, 5.8, 5.2)
    cfg = sio.default_cfg(n_rays_full=256)
    return sio.Scene(
        np.concatenate(prims), lights, np.zeros(0, sio.CLUSTER_DTYPE), np.zeros(1, np.int32),
        np.zeros(0, np.int32), np.array([0.06, 0.08, 0.12]), _camera((0, 3, 0), (-4, 1.2, -0.6), 72),
        sio.CascadeSpec((32, 16, 32), 0.45, 1), cfg,
    )


def c4_scene(n_random=50000, seed=4) -> sio.Scene:
    """SURVEY §8d C4 (unclustered): ground plane + n_random primitives."""
    ground = _prim(0, sio.PLANE, (0, 0, 0), (0, 0, 0), axis_angle((1, 0, 0), -math.pi / 2), (0.42, 0.4, 0.32))
    prims = [ground] + _random_prims(Rng(seed), n_random, 1, (-120, 0.0, -120), (120, 20.0, 120), 0.2, 2.0)
    lights = np.zeros(1, sio.LIGHT_DTYPE)
    lights[0]["kind"] = sio.LIGHT_DIRECTIONAL
    d = np.array([-0.35, -1.0, -0.25])
    lights[0]["direction"] = d / math.sqrt(float(d @ d))
    lights[0]["intensity"] = (2.6, 2.5, 2.3)
    cfg = sio.default_cfg(n_rays_full=256)
    return sio.Scene(
        np.concatenate(prims), lights, np.zeros(0, sio.CLUSTER_DTYPE), np.zeros(1, np.int32),
        np.zeros(0, np.int32), np.array([0.35, 0.45, 0.65]), _camera((0, 30, 0), (1, 29, -6), 70),
        sio.CascadeSpec((128, 32, 128), 1.875, 1), cfg,
    )


def with_fast_clusters(scene: sio.Scene, max_per_cluster=8) -> sio.Scene:
    """The scene re-clustered by the library's linear-time builder (sdfgi_build_clusters)."""
    from .runtime import build_clusters

    clusters, ms, mi = build_clusters(scene.prims, max_per_cluster)
    return sio.Scene(scene.prims, scene.lights, clusters, ms, mi, scene.sky, scene.camera, scene.cascade, scene.cfg)
