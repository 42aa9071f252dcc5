"""Renderer (pipeline.hpp:50-230) with every per-frame stage on the device.

The reference's frame loop, stage for stage, over one ``Device``:

    scene instancing + cluster build   sceneAtTime + cullAndLod (scene_file.py, host)
                                       -> sdfgi_scene_upload
    probe placement                    recenterCascade + updateProbePositions per cascade
    scheduled probe updates            selectProbesForUpdate (device) + the batched update
                                       (back atlas), budget = probe_budget or every probe
    primary visibility                 renderGBuffer (device)
    visibility + sparse GI, resolve,   sdfgi_gather against the FRONT atlas (prevField)
    contact pass
    compose                            composeFrame (device)
    roll buffers                       history on the device, atlas swap, prevCamera

``renderFrame`` returns the reference's FrameMetrics fields (stage times are
host wall-clock around each synchronous stage), ``image()`` the composed
frame; ``metrics_csv_row`` / ``write_sdfi`` write the reference's metrics.csv
rows and SDFI dumps.
"""
from __future__ import annotations

import math
import time

import numpy as np

from . import api
from . import scene_file as sf
from . import scene_io as sio
from .runtime import Device


class Renderer:
    def __init__(self, dev: Device, scene: sf.SceneFile, width: int, height: int):
        self.dev = dev
        self.file = scene
        self.cfg = scene.config.copy()
        self.width, self.height = int(width), int(height)
        self.camera = sf.buildCamera(scene.camera)
        self.prevCamera = self.camera
        self.gi = True
        self.frame = 0
        self._image = None
        cs = scene.cascade
        self.res, self.spacing0, self.levels = tuple(cs.res), float(cs.spacing), int(cs.levels)
        oct_res = int(self.cfg["oct_res"][0])
        # the scene must be on the device before the cascades (grid bounds grow over them)
        dev.upload_scene(sf.activeScene(scene, 0.0, self.camera.position))
        dev.clear_cascades()
        for level in range(self.levels):  # pipeline.hpp:61-64
            api.makeCascade(dev, *self.res, self.spacing0, level, self.camera.position, oct_res)
        dev.reset_history()

    def setCamera(self, cam: sio.Camera):
        self.camera = cam

    def setGiEnabled(self, on: bool):
        self.gi = bool(on)

    def image(self):
        """The composed frame, float64 [h, w, 3]."""
        return self._image

    def renderFrame(self) -> dict:
        dev, cfg = self.dev, self.cfg
        m = {"frame": self.frame}
        t0 = time.perf_counter()
        fps = int(cfg["fps"][0])
        active = sf.activeScene(self.file, self.frame / fps, self.camera.position)
        dev.upload_scene(active)
        m["active_primitives"], m["clusters"] = len(active.prims), len(active.clusters)
        t1 = time.perf_counter()
        rel = rej = dead = total = 0
        oct_res = int(cfg["oct_res"][0])
        for level in range(self.levels):
            res, sp, origin = dev.levels[level]
            api.recenterCascade(dev, level, *res, self.spacing0, origin, self.camera.position, oct_res)
            sp = self.spacing0 * math.pow(2.0, level)
            rep = api.updateProbePositions(dev, level, float(cfg["threshold1_frac"][0]) * sp,
                                           float(cfg["threshold2_frac"][0]) * sp,
                                           int(cfg["max_descent_steps"][0]), False, float(cfg["gradient_step"][0]))
            rel, rej, dead = rel + int(rep["relocated"]), rej + int(rep["rejected"]), dead + int(rep["dead"])
            total += dev.probe_count(level)
        m.update(relocated=rel, rejected=rej, dead=dead, probes_total=total)
        t2 = time.perf_counter()
        m["probes_updated"], m["jitter_max_texel_delta"] = 0, 0.0
        if self.gi:
            budget = int(cfg["probe_budget"][0])
            budget = budget if budget > 0 else total
            refs = None
            if budget < total:
                refs = api.selectProbesForUpdate(dev, self.camera.position, self.camera.forward, budget, self.frame)
            r = api.updateProbes(dev, cfg, self.frame, refs)
            m["probes_updated"] = min(budget, total)  # refs.size(), dead probes included (pipeline.hpp:136)
            m["jitter_max_texel_delta"] = float(r["max_texel_delta"])
        t3 = time.perf_counter()
        dev.render_gbuffer(self.camera, self.width, self.height, cfg, self.prevCamera)
        t4 = time.perf_counter()
        m["vis_traces_per_pixel"] = 0.0
        stage = [0.0, 0.0, 0.0, 0.0]
        if self.gi:
            _, vs, _ = dev.gather(self.frame, cfg, stats=True)
            m["vis_traces_per_pixel"] = int(vs["visibility_traces"]) / (self.width * self.height)
            stage = list(dev.last_gather_ms())
        else:
            dev.upload_indirect(np.zeros(3 * self.width * self.height))
        t5 = time.perf_counter()
        img, _ = dev.compose(cfg)
        t6 = time.perf_counter()
        self._image = img.reshape(self.height, self.width, 3)
        if self.gi:
            dev.swap()  # readIdx_ = writeIdx (pipeline.hpp:224)
        self.prevCamera = self.camera
        self.frame += 1
        ms = lambda a, b: (b - a) * 1e3  # noqa: E731
        gather_ms = ms(t4, t5)
        split = sum(stage)
        m.update(t_cull_ms=ms(t0, t1), t_probe_pos_ms=ms(t1, t2), t_probe_update_ms=ms(t2, t3),
                 t_gbuffer_ms=ms(t3, t4),
                 # the device gather's own stage split (visibility = downsample+select+tiles)
                 t_visibility_ms=gather_ms * (stage[0] + stage[1]) / split if split else gather_ms,
                 t_gi_resolve_ms=gather_ms * stage[2] / split if split else 0.0,
                 t_contact_ms=gather_ms * stage[3] / split if split else 0.0,
                 t_compose_ms=ms(t5, t6))
        return m
