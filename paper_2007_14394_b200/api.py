"""Reference-named host API over the C-ABI (the Python mirror of the drop-in).

Names and argument meaning follow the reference's C++ API
(/root/reference/proj/include/sdfgi/*.hpp), so callers and tests read like the
reference's own; the state they operate on lives on the GPU in a ``Device``.

    cascadeOriginFor      probe_volume.hpp:51-55
    makeCascade           probe_volume.hpp:57-76
    updateProbePositions  probe_volume.hpp:99-143
    updateProbes          batched updateProbe (probe_update.hpp:166-211) over the
                          probe stage of Renderer::renderFrame (pipeline.hpp:126-151)
    selectProbesForUpdate probe_volume.hpp:154-198 (on the device)
    recenterCascade       probe_volume.hpp:80-86
    querySceneSdf         scene.hpp:336-340
    sphereTrace           scene.hpp:391-435 (batched)
    softShadowTrace       scene.hpp:459-476 (batched)
    shadeHit              probe_update.hpp:136-149 (batched, against the front atlas)
    convolveIrradiance    probe_update.hpp:25-34 (batched over texel directions)
    interpolationStencil  probe_volume.hpp:224-310 (batched)
    composeFrame          shading.hpp:480-504 (pipeline.hpp:209)
    ProbeStage            the probe half of Renderer::renderFrame (pipeline.hpp:108-151)
"""
from __future__ import annotations

import math

import numpy as np

from . import scene_io as sio
from .runtime import Device


def snapToSpacing(p, spacing):
    """probe_volume.hpp:46-49"""
    return np.array([math.floor(x / spacing + 0.5) * spacing for x in p], dtype=np.float64)


def cascadeOriginFor(cameraPos, resX, resY, resZ, spacing):
    """probe_volume.hpp:51-55"""
    extent = np.array([(resX - 1) * spacing, (resY - 1) * spacing, (resZ - 1) * spacing])
    s = snapToSpacing(cameraPos, spacing)
    return np.array([s[i] - extent[i] * 0.5 for i in range(3)])


def makeCascade(dev: Device, resX, resY, resZ, spacing0, level, cameraPos, oct_res=8):
    """probe_volume.hpp:57-76 — allocates the cascade's probes and atlases on the device."""
    spacing = spacing0 * math.pow(2.0, level)
    origin = cascadeOriginFor(cameraPos, resX, resY, resZ, spacing)
    dev.set_cascade(level, (resX, resY, resZ), spacing, origin, oct_res)
    return level


def recenterCascade(dev: Device, level, resX, resY, resZ, spacing0, origin, cameraPos, oct_res=8):
    """probe_volume.hpp:80-86: True (and the cascade re-made: probes reset, atlases
    cleared as pipeline.hpp:110-113 does) when the snapped origin moved."""
    spacing = spacing0 * math.pow(2.0, level)
    o = cascadeOriginFor(cameraPos, resX, resY, resZ, spacing)
    if math.sqrt(float(np.dot(o - np.asarray(origin), o - np.asarray(origin)))) < 1e-12:
        return False
    dev.set_cascade(level, (resX, resY, resZ), spacing, o, oct_res)
    return True


def selectProbesForUpdate(dev: Device, cameraPos, cameraForward, budget, frameIndex):
    """probe_volume.hpp:154-198 over the device's cascades: (n, 2) int32 (cascade
    level, index) in the reference's order, n = min(budget, probes)."""
    return dev.select(cameraPos, cameraForward, budget, frameIndex)


def updateProbePositions(dev: Device, level, threshold1, threshold2, maxDescentSteps=16, stats=False,
                         gradientStep=1e-3):
    """probe_volume.hpp:99-143 (device-resident probes)."""
    return dev.relocate(level, threshold1, threshold2, maxDescentSteps, gradientStep, stats)


def updateProbes(dev: Device, cfg, frameIndex, refs=None, stats=False):
    """Batched updateProbe over `refs` ((level, index) pairs; None = all probes)."""
    return dev.update(frameIndex, cfg, refs, stats)


def composeFrame(dev: Device, cfg, indirect=None, stats=False):
    """shading.hpp:480-504 on the device's G-buffer: emission + albedo/pi * direct
    (soft-shadowed, traced on the GPU) + indirect (the last gather's contactGI
    output, or `indirect` = w*h*3 doubles). Returns the image (and TraceStats)."""
    if indirect is not None:
        dev.upload_indirect(indirect)
    r = dev.compose(cfg, stats=stats)
    return (r[0], r[2]) if stats else r[0]


def querySceneSdf(dev: Device, points, initD=None):
    """scene.hpp:336-340 at many points: (d, owner primitive index)."""
    return dev.query_points(points, initD)


def sphereTrace(dev: Device, origins, dirs, tMax, surfaceEpsilon=1e-3, maxSteps=128, startBound=math.inf):
    """scene.hpp:391-435 for a batch of rays: runtime.HIT_DTYPE records (t, pos,
    normal, prim_index, converged, miss)."""
    return dev.trace_rays(origins, dirs, tMax, surfaceEpsilon, maxSteps, startBound)


def softShadowTrace(dev: Device, origins, dirs, tMin, tMax, k, maxSteps=256, minStep=5e-4):
    """scene.hpp:459-476 for a batch of segments: visibility in [0, 1]."""
    return dev.soft_shadow(origins, dirs, tMin, tMax, k, maxSteps, minStep)


def shadeHit(dev: Device, hits, bounceCoeff, cfg):
    """probe_update.hpp:136-149 for a batch of hits (runtime.HIT_DTYPE) with the
    device's front atlas as the previous field: outgoing radiance (n, 3)."""
    return dev.shade_hits(hits, bounceCoeff, cfg)


def convolveIrradiance(dev: Device, sampleDirs, sampleRadiance, texelDirs):
    """probe_update.hpp:25-34: one sample set convolved for many directions (n, 3)."""
    return dev.convolve_irradiance(sampleDirs, sampleRadiance, texelDirs)


def interpolationStencil(dev: Device, points, mvcRelocationFrac=0.25):
    """probe_volume.hpp:224-310 over the device's cascades: runtime.STENCIL_DTYPE."""
    return dev.interpolation_stencil(points, mvcRelocationFrac)


class ProbeStage:
    """The probe half of Renderer::renderFrame (pipeline.hpp:108-151) on one device.

    Per pass: updateProbePositions for every cascade, then the batched update
    (back atlas <- front atlas, every alive probe updated with frame = pass
    index), then the frame-end swap (pipeline.hpp:220)."""

    def __init__(self, dev: Device, scene: sio.Scene, cfg=None, res=None, spacing=None, levels=None,
                 n_rays=None):
        self.dev = dev
        self.scene = scene
        self.cfg = np.array(scene.cfg if cfg is None else cfg, dtype=sio.CFG_DTYPE).reshape(1)
        if n_rays is not None:
            self.cfg["n_rays_full"] = n_rays
        self.res = tuple(scene.cascade.res if res is None else res)
        self.spacing0 = float(scene.cascade.spacing if spacing is None else spacing)
        self.levels = int(scene.cascade.levels if levels is None else levels)
        dev.upload_scene(scene)
        self.reset()

    def reset(self):
        oct_res = int(self.cfg["oct_res"][0])
        self.dev.clear_cascades()
        for level in range(self.levels):
            makeCascade(self.dev, *self.res, self.spacing0, level, self.scene.camera.position, oct_res)

    def set_scene(self, scene: sio.Scene):
        """A new frame's ActiveScene (e.g. scene_file.activeScene at the frame's time,
        pipeline.hpp:92-103) for the persistent cascades: probes and atlases keep
        their state, as in a dynamic sequence."""
        self.scene = scene
        self.dev.upload_scene(scene)

    def spacing(self, level):
        return self.spacing0 * math.pow(2.0, level)

    def relocate_all(self, stats=False):
        reps = []
        for level in range(self.levels):
            sp = self.spacing(level)
            th1 = float(self.cfg["threshold1_frac"][0]) * sp
            th2 = float(self.cfg["threshold2_frac"][0]) * sp
            reps.append(updateProbePositions(self.dev, level, th1, th2, int(self.cfg["max_descent_steps"][0]),
                                             stats, float(self.cfg["gradient_step"][0])))
        return reps

    def run_pass(self, frame, stats=False, camera=None):
        """One pass; cfg.probe_budget > 0 schedules selectProbesForUpdate's refs
        (pipeline.hpp:133-135) from `camera` (position, forward; default: the scene's).
        Without stats the pass is one sdfgi_probe_stage call (one host sync); with
        stats it keeps the per-call sequence so relocation and update counters stay
        apart."""
        budget = int(self.cfg["probe_budget"][0])
        pos = fwd = None
        if budget > 0:
            cam = self.scene.camera if camera is None else None
            pos, fwd = (cam.position, cam.forward) if cam is not None else camera
        if not stats:
            reps, upd = self.dev.probe_stage(frame, self.cfg, pos, fwd)
            self.dev.swap()
            return list(reps[:self.levels]), upd
        reps = self.relocate_all(stats)
        refs = selectProbesForUpdate(self.dev, pos, fwd, budget, frame) if budget > 0 else None
        upd = updateProbes(self.dev, self.cfg, frame, refs, stats)
        self.dev.swap()
        return reps, upd
