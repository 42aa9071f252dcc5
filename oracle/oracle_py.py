"""ctypes binding of the C oracle (oracle/sdfgi_oracle.c) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use this.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libsdfgi_oracle.so")

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    lib = ctypes.CDLL(LIB)
    sig = {
        "ora_create": ([_P, _I, _P, _I, _P, _P, _P, _I, _P], _P),
        "ora_destroy": ([_P], None),
        "ora_add_cascade": ([_P, _I, _I, _I, _I, _D, _P, _I], _I),
        "ora_relocate": ([_P, _I, _D, _D, _I, _D, _P, _P], _I),
        "ora_update": ([_P, _P, _I, _I, _I, _P, _P, _P, _P], _I),
        "ora_probes": ([_P, _I, _P, _I], _I),
        "ora_atlas": ([_P, _I, _P, ctypes.c_int64], _I),
        "ora_trace_rays": ([_P, _P, _I, _I, _I, _P, _I], _I),
        "ora_query": ([_P, _P, _P, _I, _P, _P], None),
        "ora_render_gbuffer": ([_P, _P, _I, _I, _P, _P, _P], _I),
        "ora_gather_frame": ([_P, _P, _I, _I, _I, _P, _P, _P, _I] + [_P] * 10, _I),
        "ora_compose": ([_P, _P, _I, _I, _P, _P, _P, _P], _I),
        "ora_select": ([_P, _P, _P, _I, _I, _P], _I),
        "ora_update_refs": ([_P, _P, _I, _P, _I, _I, _P, _P, _P, _P], _I),
        "ora_set_threads": ([_I], None),
        "ora_atlas_set": ([_P, _I, _P, ctypes.c_int64], _I),
        "ora_mark_updated": ([_P, _P, _I, _I], _I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    # the gather's row loops and renderGBuffer on every host core (results do not
    # depend on the thread count: each row is independent, statistics are summed)
    lib.ora_set_threads(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    _lib = lib
    return lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _origin(cam, res, spacing):
    """cascadeOriginFor (probe_volume.hpp:51-55)."""
    return np.array([math.floor(cam[i] / spacing + 0.5) * spacing - ((res[i] - 1) * spacing) * 0.5 for i in range(3)])


class Stage:
    """The reference probe stage restated in C: scene + cascades + front/back atlases."""

    def __init__(self, scene, cfg=None, res=None, spacing=None, levels=None):
        from paper_2007_14394_b200 import scene_io as sio

        self.sio = sio
        lib = load()
        self.scene = scene
        self.cfg = np.array(scene.cfg if cfg is None else cfg, dtype=sio.CFG_DTYPE).reshape(1)
        self._keep = [np.ascontiguousarray(x) for x in (scene.prims, scene.clusters, scene.member_start,
                                                        scene.member_idx, scene.lights, scene.sky)]
        pr, cl, ms, mi, li, sky = self._keep
        self.h = lib.ora_create(_p(pr), len(pr), _p(cl), len(cl), _p(ms.astype(np.int32)), _p(mi.astype(np.int32)),
                                _p(li), len(li), _p(sky.astype(np.float64)))
        self.res = tuple(scene.cascade.res if res is None else res)
        self.spacing0 = float(scene.cascade.spacing if spacing is None else spacing)
        self.levels = int(scene.cascade.levels if levels is None else levels)
        oct_res = int(self.cfg["oct_res"][0])
        for level in range(self.levels):
            sp = self.spacing0 * math.pow(2.0, level)
            o = _origin(scene.camera.position, self.res, sp)
            lib.ora_add_cascade(self.h, level, *self.res, sp, _p(o), oct_res)
        self.oct = oct_res

    def close(self):
        if getattr(self, "h", None):
            load().ora_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def spacing(self, level):
        return self.spacing0 * math.pow(2.0, level)

    def relocate_all(self):
        reps, stats = [], np.zeros(8, np.uint64)
        for level in range(self.levels):
            sp = self.spacing(level)
            rep = np.zeros(3, np.int32)
            load().ora_relocate(self.h, level, float(self.cfg["threshold1_frac"][0]) * sp,
                                float(self.cfg["threshold2_frac"][0]) * sp, int(self.cfg["max_descent_steps"][0]),
                                float(self.cfg["gradient_step"][0]), _p(rep), _p(stats))
            reps.append(rep)
        return reps, stats

    def update(self, frame, stride=1, threads=1):
        md = ctypes.c_double()
        rays, upd = ctypes.c_int64(), ctypes.c_int64()
        stats = np.zeros(8, np.uint64)
        rc = load().ora_update(self.h, _p(self.cfg), frame, stride, threads, ctypes.byref(md), ctypes.byref(rays),
                               ctypes.byref(upd), _p(stats))
        assert rc == 0
        return md.value, rays.value, upd.value, stats

    def select(self, budget, frame, cam_pos=None, cam_fwd=None):
        """selectProbesForUpdate (probe_volume.hpp:154-198) -> (n, 2) int32 (slot, index)."""
        cp = np.ascontiguousarray(self.scene.camera.position if cam_pos is None else cam_pos, np.float64)
        cf = np.ascontiguousarray(self.scene.camera.forward if cam_fwd is None else cam_fwd, np.float64)
        out = np.zeros((max(budget, 0), 2), np.int32)
        n = load().ora_select(self.h, _p(cp), _p(cf), int(budget), int(frame), _p(out))
        return out[:n]

    def update_refs(self, frame, refs, threads=1):
        refs = np.ascontiguousarray(refs, np.int32).reshape(-1, 2)
        md = ctypes.c_double()
        rays, upd = ctypes.c_int64(), ctypes.c_int64()
        stats = np.zeros(8, np.uint64)
        rc = load().ora_update_refs(self.h, _p(self.cfg), frame, _p(refs), len(refs), threads, ctypes.byref(md),
                                    ctypes.byref(rays), ctypes.byref(upd), _p(stats))
        assert rc == 0
        return md.value, rays.value, upd.value, stats

    def run_pass(self, frame, stride=1, threads=1):
        reps, rstats = self.relocate_all()
        return reps, rstats, self.update(frame, stride, threads)

    def probes(self, level):
        n = self.res[0] * self.res[1] * self.res[2]
        out = np.zeros(n, self.sio.PROBE_DTYPE)
        assert load().ora_probes(self.h, level, _p(out), n) == 0
        return out

    def atlas(self, level):
        n = self.res[0] * self.res[1] * self.res[2]
        t = self.oct + 2
        out = np.zeros((n, t, t, 3), np.float32)
        assert load().ora_atlas(self.h, level, _p(out), out.size) == 0
        return out

    def set_atlas(self, level, atlas):
        """Overwrite the front atlas of a cascade (test hook: the slab exchange)."""
        a = np.ascontiguousarray(atlas, np.float32)
        assert load().ora_atlas_set(self.h, level, _p(a), a.size) == 0

    def mark_updated(self, frame, refs):
        """rejectHistory = false, lastUpdateFrame = frame for the alive probes of refs
        (probe_update.hpp:208-209) without tracing them (test hook)."""
        r = np.ascontiguousarray(refs, np.int32).reshape(-1, 2)
        assert load().ora_mark_updated(self.h, _p(r), len(r), frame) == 0

    def trace_rays(self, frame, probe, level=0):
        cap = 2 * int(self.cfg["n_rays_full"][0])
        out = np.zeros(cap, self.sio.RAY_DTYPE)
        n = load().ora_trace_rays(self.h, _p(self.cfg), frame, level, probe, _p(out), cap)
        assert n >= 0
        return out[:n]

    def camera(self):
        c = self.scene.camera
        cam = np.zeros(1, self.sio.CAMERA_DTYPE)
        cam["position"], cam["forward"], cam["right"], cam["up"] = c.position, c.forward, c.right, c.up
        cam["fov_y_deg"] = c.fov_y
        return cam

    def render_gbuffer(self, w, h):
        out = np.zeros(w * h, self.sio.GBUFFER_DTYPE)
        stats = np.zeros(8, np.uint64)
        load().ora_render_gbuffer(self.h, _p(self.camera()), w, h, _p(self.cfg), _p(out), _p(stats))
        return out, stats

    def gather_frame(self, gb, w, h, frame, hist=None):
        """One gather frame (pipeline.hpp:161-207); hist = (resolved[w*h*3], depth[w*h]) or None."""
        hw, hh = (w + 1) // 2, (h + 1) // 2
        sw, sh = (hw + 1) // 2, (hh + 1) // 2
        out = dict(half_depth=np.zeros(hw * hh), half_src=np.zeros(hw * hh, np.int32),
                   sel=np.zeros(sw * sh, np.int32), sparse_irr=np.zeros(sw * sh * 3),
                   sparse_valid=np.zeros(sw * sh, np.int32), sparse_anchor=np.zeros(sw * sh, np.int32),
                   resolved=np.zeros(w * h * 3), indirect=np.zeros(w * h * 3),
                   vis_stats=np.zeros(8, np.uint64), contact_stats=np.zeros(8, np.uint64))
        gb = np.ascontiguousarray(gb, self.sio.GBUFFER_DTYPE)
        hi = None if hist is None else np.ascontiguousarray(hist[0], np.float64)
        hd = None if hist is None else np.ascontiguousarray(hist[1], np.float64)
        n = load().ora_gather_frame(self.h, _p(gb), w, h, frame, _p(self.cfg), _p(hi), _p(hd),
                                    0 if hist is None else 1, *[_p(out[k]) for k in (
                                        "half_depth", "half_src", "sel", "sparse_irr", "sparse_valid",
                                        "sparse_anchor", "resolved", "indirect", "vis_stats", "contact_stats")])
        out["tasks"] = n
        return out

    def compose(self, gb, w, h, indirect):
        """composeFrame (shading.hpp:480-504): the final image, 3 doubles per pixel."""
        gb = np.ascontiguousarray(gb, self.sio.GBUFFER_DTYPE)
        ind = np.ascontiguousarray(indirect, np.float64)
        out = np.zeros(w * h * 3)
        stats = np.zeros(8, np.uint64)
        load().ora_compose(self.h, _p(gb), w, h, _p(ind), _p(self.cfg), _p(out), _p(stats))
        return out, stats

    def query(self, pts, init=None):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        ini = None if init is None else np.ascontiguousarray(init, np.float64)
        d = np.zeros(len(pts))
        o = np.zeros(len(pts), np.int32)
        load().ora_query(self.h, _p(pts), _p(ini), len(pts), _p(d), _p(o))
        return d, o
