"""ctypes binding of libsdfgi_b200.so (the C-ABI in include/sdfgi_b200.h).

This is the Python-side view of the drop-in boundary. It never falls back to a
CPU path: if the library is missing or no CUDA device exists, constructing a
``Device`` raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import scene_io as sio

_PKG = os.path.dirname(os.path.abspath(__file__))
# SDFGI_LIB: load another build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("SDFGI_LIB") or os.path.join(_PKG, "libsdfgi_b200.so")

F64, F32 = 0, 1
_PREC = {"f64": F64, "f32": F32, F64: F64, F32: F32}

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> argtypes (restype int unless noted)
_SIGS = {
    "sdfgi_abi_version": [],
    "sdfgi_last_error": [],
    "sdfgi_device_count": [_P],
    "sdfgi_nccl_unique_id": [_P],
    "sdfgi_ctx_create": [_I, _I, _I, _P, _I, _P],
    "sdfgi_ctx_destroy": [_P],
    "sdfgi_ctx_set_precision": [_P, _I],
    "sdfgi_ctx_stream": [_P, _P],
    "sdfgi_ctx_synchronize": [_P],
    "sdfgi_scene_upload": [_P, _P, _I, _P, _I, _P, _P, _P, _I, _P],
    "sdfgi_lights_upload": [_P, _P, _I, _P],
    "sdfgi_cascade_set": [_P, _I, _I, _I, _I, _D, _P, _I],
    "sdfgi_cascade_count": [_P, _P],
    "sdfgi_cascades_clear": [_P],
    "sdfgi_probes_reset": [_P, _I],
    "sdfgi_probes_upload": [_P, _I, _P, _I],
    "sdfgi_probes_download": [_P, _I, _P, _I],
    "sdfgi_probes_relocate": [_P, _I, _D, _D, _I, _D, _P, _P],
    "sdfgi_probes_update": [_P, _P, _I, _I, _P, _P, _P],
    "sdfgi_probe_stage": [_P, _I, _P, _P, _P, _P, _I, _P, _P],
    "sdfgi_stage_ms_sum": [_P, _P, _I],
    "sdfgi_probe_stage_async": [_P, _I, _P, _P, _P],
    "sdfgi_probe_stage_collect": [_P, _P, _I, _P, _I, _P],
    "sdfgi_atlas_swap": [_P],
    "sdfgi_atlas_download": [_P, _I, _I, _P, _SZ],
    "sdfgi_atlas_upload": [_P, _I, _I, _P, _SZ],
    "sdfgi_atlas_device_ptr": [_P, _I, _I, _P, _P],
    "sdfgi_probes_trace_debug": [_P, _P, _I, _I, _P, _P, _I, _P],
    "sdfgi_query_points": [_P, _P, _P, _I, _P, _P],
    "sdfgi_last_kernel_ms": [_P, _P, _P],
    "sdfgi_last_work": [_P, _P],
    "sdfgi_last_shading_work": [_P, _P],
    "sdfgi_last_stage_ms": [_P, _P],
    "sdfgi_last_trace_counters": [_P, _P],
    "sdfgi_measure_fp_peak": [_P, _P, _P],
    "sdfgi_set_accel": [_P, _I],
    "sdfgi_accel_info": [_P, _P],
    "sdfgi_slab_range": [_I, _I, _I, _I, _I, _P, _P],
    "sdfgi_build_clusters": [_P, _I, _I, _P, _P, _P, _P],
    "sdfgi_gbuffer_upload": [_P, _I, _I, _P],
    "sdfgi_gbuffer_render": [_P, _P, _P, _I, _I, _P],
    "sdfgi_gbuffer_download": [_P, _P, _SZ],
    "sdfgi_gather": [_P, _I, _P, _P, _P, _P],
    "sdfgi_gather_reset_history": [_P],
    "sdfgi_gather_download": [_P, _I, _P, _SZ],
    "sdfgi_last_gather_ms": [_P, _P],
    "sdfgi_indirect_upload": [_P, _P, _SZ],
    "sdfgi_compose": [_P, _P, _P, _P],
    "sdfgi_select_probes": [_P, _P, _P, _I, _I, _P, _P],
    "sdfgi_launch_count": [_P, _P],
    "sdfgi_trace_rays": [_P, _P, _P, _I, _D, _D, _I, _D, _P, _P],
    "sdfgi_soft_shadow": [_P, _P, _P, _P, _P, _I, _D, _I, _D, _P, _P],
    "sdfgi_shade_hits": [_P, _P, _I, _D, _P, _P, _P],
    "sdfgi_convolve_irradiance": [_P, _P, _P, _I, _P, _I, _P],
    "sdfgi_interpolation_stencil": [_P, _P, _I, _D, _P],
}

# sdfgi_hit (Hit, scene.hpp:375-383) and sdfgi_stencil (InterpolationStencil,
# probe_volume.hpp:205-217), include/sdfgi_b200.h
HIT_DTYPE = np.dtype([("t", "<f8"), ("pos", "<f8", 3), ("normal", "<f8", 3), ("prim_index", "<i4"),
                      ("converged", "<i4"), ("miss", "<i4"), ("_pad", "<i4")])
STENCIL_DTYPE = np.dtype([("weight", "<f8", 8), ("level", "<i4"), ("index", "<i4", 8), ("count", "<i4"),
                          ("cross_cascade", "<i4"), ("sky_fallback", "<i4"), ("used_mvc", "<i4"), ("_pad", "<i4")])

RELOC_DTYPE = np.dtype([("relocated", "<i4"), ("rejected", "<i4"), ("dead", "<i4"), ("_pad", "<i4")])
RESULT_DTYPE = np.dtype([("max_texel_delta", "<f8"), ("rays_traced", "<i8"), ("probes_updated", "<i8")])

_lib = None


class SdfgiError(RuntimeError):
    def __init__(self, fn, code, msg):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


def load_library(path: str = LIB_PATH):
    """Load the CUDA library (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2007_14394_b200.build` "
            "(the B200 path has no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_char_p if name == "sdfgi_last_error" else ctypes.c_int
    _lib = lib
    return lib


def exported_symbols():
    return list(_SIGS)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _call(name, *args):
    lib = load_library()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise SdfgiError(name, rc, lib.sdfgi_last_error().decode())
    return rc


def camera_struct(cam) -> np.ndarray:
    """scene_io.Camera -> sdfgi_camera (1-element array)."""
    c = np.zeros(1, sio.CAMERA_DTYPE)
    c["position"], c["forward"], c["right"], c["up"] = cam.position, cam.forward, cam.right, cam.up
    c["fov_y_deg"] = cam.fov_y
    return c


def build_clusters(prims, max_per_cluster=8):
    """Linear-time cluster build (sdfgi_build_clusters): (clusters, member_start, member_idx)."""
    prims = np.ascontiguousarray(prims, sio.PRIM_DTYPE)
    n = len(prims)
    clusters = np.zeros(max(n, 1), sio.CLUSTER_DTYPE)
    ms = np.zeros(n + 1, np.int32)
    mi = np.zeros(max(n, 1), np.int32)
    k = ctypes.c_int()
    _call("sdfgi_build_clusters", _ptr(prims), n, int(max_per_cluster), _ptr(clusters), ctypes.byref(k), _ptr(ms),
          _ptr(mi))
    return clusters[: k.value].copy(), ms[: k.value + 1].copy(), mi[:n].copy()


def device_count() -> int:
    n = ctypes.c_int(0)
    _call("sdfgi_device_count", ctypes.byref(n))
    return n.value


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _call("sdfgi_nccl_unique_id", buf)
    return bytes(buf)


class Device:
    """One context on one GPU (one rank of a slab-sharded job when world > 1)."""

    def __init__(self, device=0, rank=0, world=1, nccl_uid: bytes | None = None, precision="f64"):
        self._ctx = ctypes.c_void_p()
        uid = None
        if nccl_uid is not None:
            uid = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_uid)
        _call("sdfgi_ctx_create", device, rank, world, uid, _PREC[precision], ctypes.byref(self._ctx))
        self.rank, self.world, self.device = rank, world, device
        self.precision = precision
        self.levels = {}  # level -> (res, spacing, origin)
        self.oct_res = 8

    def close(self):
        if self._ctx:
            load_library().sdfgi_ctx_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------- context
    def set_precision(self, precision):
        _call("sdfgi_ctx_set_precision", self._ctx, _PREC[precision])
        self.precision = precision

    @property
    def stream(self) -> int:
        s = ctypes.c_void_p()
        _call("sdfgi_ctx_stream", self._ctx, ctypes.byref(s))
        return s.value or 0

    def synchronize(self):
        _call("sdfgi_ctx_synchronize", self._ctx)

    def last_kernel_ms(self):
        """(update kernel ms, relocation kernel ms) of the most recent launches."""
        a, b = ctypes.c_double(), ctypes.c_double()
        _call("sdfgi_last_kernel_ms", self._ctx, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def last_shading_work(self):
        """(shadeHit calls, MVC evaluations) of the last stats-enabled update."""
        out = np.zeros(2, np.uint64)
        _call("sdfgi_last_shading_work", self._ctx, _ptr(out))
        return int(out[0]), int(out[1])

    STAGES = ("k1", "k1_far", "normals", "k2", "k2_far", "shade", "convolve")

    def last_stage_ms(self):
        """Device ms of the last update's stages (CUDA events on the context's stream):
        dict over STAGES (K1, its far phase, compaction + normals, K2, its far phase,
        K3a + K3c, K3b)."""
        out = np.zeros(7)
        _call("sdfgi_last_stage_ms", self._ctx, _ptr(out))
        return dict(zip(self.STAGES, map(float, out)))

    def stage_ms_sum(self, reset=True):
        """Stage ms summed over the updates since the last reset: (dict over STAGES,
        the updates' total ms)."""
        out = np.zeros(8)
        _call("sdfgi_stage_ms_sum", self._ctx, _ptr(out), 1 if reset else 0)
        return dict(zip(self.STAGES, map(float, out[:7]))), float(out[7])

    def last_trace_counters(self):
        """The last stats-enabled update's counters per tracing kernel: {"k1": ..., "k2": ...},
        each (stats dict, evaluations by kind x5 + rotated)."""
        out = np.zeros(28, np.uint64)
        _call("sdfgi_last_trace_counters", self._ctx, _ptr(out))
        names = ("sdf_queries", "clusters_visited", "clusters_skipped", "primitive_evals", "trace_steps",
                 "sphere_traces", "shadow_traces", "visibility_traces")
        res = {}
        for k, key in enumerate(("k1", "k2")):
            v = [int(x) for x in out[14 * k:14 * k + 14]]
            res[key] = (dict(zip(names, v[:8])), v[8:])
        return res

    def last_work(self):
        """Evaluations by kind (sphere, box, plane, cylinder, capsule, rotated) of the last
        stats-enabled call."""
        out = np.zeros(6, np.uint64)
        _call("sdfgi_last_work", self._ctx, _ptr(out))
        return out

    def measure_fp_peak(self):
        """(FP64 FMA/s, FP32 FMA/s) measured on this device."""
        a, b = ctypes.c_double(), ctypes.c_double()
        _call("sdfgi_measure_fp_peak", self._ctx, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def set_accel(self, mode: int):
        """0: the reference's flat cluster walk (exact TraceStats); 1: candidate grid (the
        exact march sequence, query counts equal to the reference's); 2 (default): grid,
        and marches that leave the grid box for good end as misses at once (outputs
        unchanged, fewer queries)."""
        _call("sdfgi_set_accel", self._ctx, int(mode))

    def accel_info(self):
        out = np.zeros(6, np.int64)
        _call("sdfgi_accel_info", self._ctx, _ptr(out))
        return {"mode": int(out[0]), "grid": bool(out[1]), "dim": tuple(int(x) for x in out[2:5]),
                "entries": int(out[5])}

    # ---------------------------------------------------------- gather (e)
    def upload_gbuffer(self, w, h, pixels):
        px = np.ascontiguousarray(pixels, sio.GBUFFER_DTYPE)
        assert len(px) == w * h
        _call("sdfgi_gbuffer_upload", self._ctx, int(w), int(h), _ptr(px))
        self.gsize = (int(w), int(h))

    def render_gbuffer(self, camera, w, h, cfg, prev_camera=None):
        cam = camera_struct(camera)
        prev = None if prev_camera is None else camera_struct(prev_camera)
        cfg = np.ascontiguousarray(cfg, sio.CFG_DTYPE)
        _call("sdfgi_gbuffer_render", self._ctx, _ptr(cam), _ptr(prev), int(w), int(h), _ptr(cfg))
        self.gsize = (int(w), int(h))

    def gbuffer(self):
        w, h = self.gsize
        out = np.zeros(w * h, sio.GBUFFER_DTYPE)
        _call("sdfgi_gbuffer_download", self._ctx, _ptr(out), out.size)
        return out

    def gather(self, frame, cfg, stats=False):
        """One gather frame; returns the number of visibility tasks (and stats)."""
        cfg = np.ascontiguousarray(cfg, sio.CFG_DTYPE)
        n = ctypes.c_int64()
        vs = np.zeros(1, sio.STATS_DTYPE) if stats else None
        cs = np.zeros(1, sio.STATS_DTYPE) if stats else None
        _call("sdfgi_gather", self._ctx, int(frame), _ptr(cfg), ctypes.byref(n), _ptr(vs), _ptr(cs))
        return (n.value, vs[0], cs[0]) if stats else n.value

    def reset_history(self):
        _call("sdfgi_gather_reset_history", self._ctx)

    def upload_indirect(self, rgb):
        a = np.ascontiguousarray(rgb, np.float64).reshape(-1)
        _call("sdfgi_indirect_upload", self._ctx, _ptr(a), a.size)

    def compose(self, cfg, stats=False, download=True):
        """composeFrame (shading.hpp:480-504) on the context's G-buffer and indirect
        image; returns (image[w*h*3] or None, device ms[, stats])."""
        c = np.ascontiguousarray(cfg, sio.CFG_DTYPE)
        st = np.zeros(1, sio.STATS_DTYPE) if stats else None
        ms = np.zeros(1)
        _call("sdfgi_compose", self._ctx, _ptr(c), _ptr(st), _ptr(ms))
        img = self.gather_buffer("composed") if download else None
        return (img, float(ms[0]), st[0]) if stats else (img, float(ms[0]))

    def gather_buffer(self, name):
        w, h = self.gsize
        hw, hh = (w + 1) // 2, (h + 1) // 2
        sw, sh = (hw + 1) // 2, (hh + 1) // 2
        spec = {"resolved": (0, w * h * 3, np.float64), "indirect": (1, w * h * 3, np.float64),
                "half_depth": (2, hw * hh, np.float64), "half_src": (3, hw * hh, np.int32),
                "sel": (4, sw * sh, np.int32), "sparse_irr": (5, sw * sh * 3, np.float64),
                "sparse_valid": (6, sw * sh, np.int32), "sparse_anchor": (7, sw * sh, np.int32),
                "composed": (8, w * h * 3, np.float64)}
        which, n, dt = spec[name]
        out = np.zeros(n, dt)
        _call("sdfgi_gather_download", self._ctx, which, _ptr(out), out.nbytes)
        return out

    def last_gather_ms(self):
        out = np.zeros(4)
        _call("sdfgi_last_gather_ms", self._ctx, _ptr(out))
        return out

    def launch_count(self) -> int:
        n = ctypes.c_int64()
        _call("sdfgi_launch_count", self._ctx, ctypes.byref(n))
        return n.value

    # --------------------------------------------------------------- scene
    def upload_scene(self, s: sio.Scene):
        prims = np.ascontiguousarray(s.prims, sio.PRIM_DTYPE)
        clusters = np.ascontiguousarray(s.clusters, sio.CLUSTER_DTYPE)
        ms = np.ascontiguousarray(s.member_start, np.int32)
        mi = np.ascontiguousarray(s.member_idx, np.int32)
        lights = np.ascontiguousarray(s.lights, sio.LIGHT_DTYPE)
        sky = np.ascontiguousarray(s.sky, np.float64)
        _call("sdfgi_scene_upload", self._ctx, _ptr(prims), len(prims), _ptr(clusters), len(clusters),
              _ptr(ms), _ptr(mi), _ptr(lights), len(lights), _ptr(sky))

    def upload_lights(self, lights, sky):
        lights = np.ascontiguousarray(lights, sio.LIGHT_DTYPE)
        sky = np.ascontiguousarray(sky, np.float64)
        _call("sdfgi_lights_upload", self._ctx, _ptr(lights), len(lights), _ptr(sky))

    # -------------------------------------------------------------- probes
    def set_cascade(self, level, res, spacing, origin, oct_res=8):
        o = np.ascontiguousarray(origin, np.float64)
        _call("sdfgi_cascade_set", self._ctx, level, int(res[0]), int(res[1]), int(res[2]), float(spacing),
              _ptr(o), oct_res)
        self.levels[level] = (tuple(int(r) for r in res), float(spacing), o.copy())
        self.oct_res = oct_res

    def clear_cascades(self):
        _call("sdfgi_cascades_clear", self._ctx)
        self.levels = {}

    def probe_count(self, level) -> int:
        r = self.levels[level][0]
        return r[0] * r[1] * r[2]

    def reset_probes(self, level):
        _call("sdfgi_probes_reset", self._ctx, level)

    def probes(self, level) -> np.ndarray:
        out = np.zeros(self.probe_count(level), sio.PROBE_DTYPE)
        _call("sdfgi_probes_download", self._ctx, level, _ptr(out), len(out))
        return out

    def upload_probes(self, level, probes):
        p = np.ascontiguousarray(probes, sio.PROBE_DTYPE)
        _call("sdfgi_probes_upload", self._ctx, level, _ptr(p), len(p))

    def relocate(self, level, th1, th2, max_steps=16, grad_step=1e-3, stats=False):
        rep = np.zeros(1, RELOC_DTYPE)
        st = np.zeros(1, sio.STATS_DTYPE) if stats else None
        _call("sdfgi_probes_relocate", self._ctx, level, float(th1), float(th2), int(max_steps),
              float(grad_step), _ptr(rep), _ptr(st))
        return (rep[0], st[0]) if stats else rep[0]

    def update(self, frame, cfg, refs=None, stats=False):
        """refs: None (all probes) or an int array of (level, index) pairs."""
        cfg = np.ascontiguousarray(cfg, sio.CFG_DTYPE)
        res = np.zeros(1, RESULT_DTYPE)
        st = np.zeros(1, sio.STATS_DTYPE) if stats else None
        r = None if refs is None else np.ascontiguousarray(refs, np.int32).reshape(-1, 2)
        _call("sdfgi_probes_update", self._ctx, _ptr(r), 0 if r is None else len(r), int(frame), _ptr(cfg),
              _ptr(res), _ptr(st))
        return (res[0], st[0]) if stats else res[0]

    def probe_stage(self, frame, cfg, cam_pos=None, cam_fwd=None, stats=False):
        """Relocation of every cascade + (budgeted) selection + update in one call
        (sdfgi_probe_stage): -> (reports per cascade, result[, stats])."""
        cfg = np.ascontiguousarray(cfg, sio.CFG_DTYPE)
        reps = np.zeros(max(len(self.levels), 1), RELOC_DTYPE)  # cascade creation order
        res = np.zeros(1, RESULT_DTYPE)
        st = np.zeros(1, sio.STATS_DTYPE) if stats else None
        cp = None if cam_pos is None else np.ascontiguousarray(cam_pos, np.float64)
        cf = None if cam_fwd is None else np.ascontiguousarray(cam_fwd, np.float64)
        _call("sdfgi_probe_stage", self._ctx, int(frame), _ptr(cfg), _ptr(cp), _ptr(cf), _ptr(reps), len(reps),
              _ptr(res), _ptr(st))
        return (reps, res[0], st[0]) if stats else (reps, res[0])

    def probe_stage_async(self, frame, cfg, cam_pos=None, cam_fwd=None):
        """Queue one probe stage pass (sdfgi_probe_stage_async) and return at once."""
        cfg = np.ascontiguousarray(cfg, sio.CFG_DTYPE)
        cp = None if cam_pos is None else np.ascontiguousarray(cam_pos, np.float64)
        cf = None if cam_fwd is None else np.ascontiguousarray(cam_fwd, np.float64)
        _call("sdfgi_probe_stage_async", self._ctx, int(frame), _ptr(cfg), _ptr(cp), _ptr(cf))

    def probe_stage_collect(self, max_passes=8):
        """Wait for the queued passes -> (reports [passes, cascades], results [passes])."""
        nc = max(len(self.levels), 1)
        reps = np.zeros((max_passes, nc), RELOC_DTYPE)
        res = np.zeros(max_passes, RESULT_DTYPE)
        n = ctypes.c_int()
        _call("sdfgi_probe_stage_collect", self._ctx, _ptr(reps), nc, _ptr(res), max_passes, ctypes.byref(n))
        return reps[:n.value], res[:n.value]

    def select(self, cam_pos, cam_fwd, budget, frame):
        """selectProbesForUpdate on the device -> (n, 2) int32 (level, index)."""
        cp = np.ascontiguousarray(cam_pos, np.float64)
        cf = np.ascontiguousarray(cam_fwd, np.float64)
        out = np.zeros((max(int(budget), 0), 2), np.int32)
        n = ctypes.c_int()
        _call("sdfgi_select_probes", self._ctx, _ptr(cp), _ptr(cf), int(budget), int(frame), _ptr(out),
              ctypes.byref(n))
        return out[:n.value]

    def swap(self):
        _call("sdfgi_atlas_swap", self._ctx)

    def atlas(self, level, which=0, out=None) -> np.ndarray:
        """which 0 = front (read) atlas, 1 = back (write). Shape [P, R+2, R+2, 3].
        out: a C-contiguous float32 array of that size (e.g. pinned) to download into."""
        t = self.oct_res + 2
        shape = (self.probe_count(level), t, t, 3)
        if out is None:
            out = np.zeros(shape, np.float32)
        elif out.dtype != np.float32 or not out.flags.c_contiguous or out.size != int(np.prod(shape)):
            raise ValueError("atlas out: C-contiguous float32 array of %s expected" % (shape,))
        _call("sdfgi_atlas_download", self._ctx, level, which, _ptr(out), out.size)
        return out

    def upload_atlas(self, level, data, which=0):
        a = np.ascontiguousarray(data, np.float32)
        _call("sdfgi_atlas_upload", self._ctx, level, which, _ptr(a), a.size)

    def atlas_device_ptr(self, level, which=0):
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _call("sdfgi_atlas_device_ptr", self._ctx, level, which, ctypes.byref(p), ctypes.byref(n))
        return p.value, n.value

    def trace_debug(self, frame, cfg, refs):
        cfg = np.ascontiguousarray(cfg, sio.CFG_DTYPE)
        r = np.ascontiguousarray(refs, np.int32).reshape(-1, 2)
        cap = len(r) * 2 * int(cfg["n_rays_full"][0])
        out = np.zeros(cap, sio.RAY_DTYPE)
        n = ctypes.c_int()
        _call("sdfgi_probes_trace_debug", self._ctx, _ptr(r), len(r), int(frame), _ptr(cfg), _ptr(out), cap,
              ctypes.byref(n))
        return out[: n.value]

    def trace_rays(self, origins, dirs, t_max, eps=1e-3, max_steps=128, start_bound=np.inf, stats=False):
        """sphereTrace (scene.hpp:391-435) of a batch of rays -> HIT_DTYPE array."""
        o = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
        out = np.zeros(len(o), HIT_DTYPE)
        st = np.zeros(1, sio.STATS_DTYPE) if stats else None
        _call("sdfgi_trace_rays", self._ctx, _ptr(o), _ptr(d), len(o), float(t_max), float(eps), int(max_steps),
              float(start_bound), _ptr(out), _ptr(st))
        return (out, st[0]) if stats else out

    def soft_shadow(self, origins, dirs, t_min, t_max, k, max_steps=256, min_step=5e-4, stats=False):
        """softShadowTrace (scene.hpp:459-476) of a batch of segments -> visibility."""
        o = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
        t0 = np.ascontiguousarray(np.broadcast_to(t_min, len(o)), np.float64)
        t1 = np.ascontiguousarray(np.broadcast_to(t_max, len(o)), np.float64)
        v = np.zeros(len(o))
        st = np.zeros(1, sio.STATS_DTYPE) if stats else None
        _call("sdfgi_soft_shadow", self._ctx, _ptr(o), _ptr(d), _ptr(t0), _ptr(t1), len(o), float(k), int(max_steps),
              float(min_step), _ptr(v), _ptr(st))
        return (v, st[0]) if stats else v

    def shade_hits(self, hits, bounce_coeff, cfg):
        """shadeHit (probe_update.hpp:136-149) of HIT_DTYPE hits against the front atlas."""
        h = np.ascontiguousarray(hits, HIT_DTYPE)
        c = np.ascontiguousarray(cfg, sio.CFG_DTYPE).reshape(1)
        out = np.zeros((len(h), 3))
        _call("sdfgi_shade_hits", self._ctx, _ptr(h), len(h), float(bounce_coeff), _ptr(c), _ptr(out), None)
        return out

    def convolve_irradiance(self, sample_dirs, sample_radiance, texel_dirs):
        """convolveIrradiance (probe_update.hpp:25-34) for many texel directions."""
        sd = np.ascontiguousarray(sample_dirs, np.float64).reshape(-1, 3)
        sr = np.ascontiguousarray(sample_radiance, np.float64).reshape(-1, 3)
        td = np.ascontiguousarray(texel_dirs, np.float64).reshape(-1, 3)
        out = np.zeros((len(td), 3))
        _call("sdfgi_convolve_irradiance", self._ctx, _ptr(sd), _ptr(sr), len(sd), _ptr(td), len(td), _ptr(out))
        return out

    def interpolation_stencil(self, points, mvc_frac=0.25):
        """interpolationStencil (probe_volume.hpp:224-310) -> STENCIL_DTYPE array."""
        p = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        out = np.zeros(len(p), STENCIL_DTYPE)
        _call("sdfgi_interpolation_stencil", self._ctx, _ptr(p), len(p), float(mvc_frac), _ptr(out))
        return out

    def query_points(self, pts, init=None):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        ini = None if init is None else np.ascontiguousarray(init, np.float64)
        d = np.zeros(len(pts))
        o = np.zeros(len(pts), np.int32)
        _call("sdfgi_query_points", self._ctx, _ptr(pts), _ptr(ini), len(pts), _ptr(d), _ptr(o))
        return d, o
