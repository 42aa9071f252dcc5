"""SDFS scene interchange file and the numpy mirrors of the C-ABI structs.

The structs in ``include/sdfgi_b200.h`` are both the ABI and the on-disk layout.
An SDFS file is what the reference's scene loader produces after
``sceneAtTime`` + ``cullAndLod`` (scene_file.hpp:584-645, scene.hpp:188-203):
instanced primitives, lights, sky, and the cluster cull bounds + CSR member
lists (``QueryAccel``, scene.hpp:50-86). Both the reference driver
(oracle/ref_driver.cpp) and this package read and write it, so the CPU
reference and the GPU path see byte-identical inputs.

Layout: 176-byte header, ``sdfgi_cfg`` (224 B), prims (184 B each), lights
(80 B), clusters (56 B), int32 member_start[K+1], int32 member_idx[M], padded
to 8 bytes.
"""
from __future__ import annotations

import dataclasses
import struct

import numpy as np

PRIM_DTYPE = np.dtype(
    [
        ("id", "<i4"),
        ("kind", "<i4"),
        ("lod_tier", "<i4"),
        ("_pad", "<i4"),
        ("rot", "<f8", (9,)),
        ("trans", "<f8", (3,)),
        ("size", "<f8", (3,)),
        ("albedo", "<f8", (3,)),
        ("emission", "<f8", (3,)),
    ]
)
LIGHT_DTYPE = np.dtype(
    [
        ("kind", "<i4"),
        ("_pad", "<i4"),
        ("position", "<f8", (3,)),
        ("direction", "<f8", (3,)),
        ("intensity", "<f8", (3,)),
    ]
)
CLUSTER_DTYPE = np.dtype(
    [("lo", "<f8", (3,)), ("hi", "<f8", (3,)), ("unbounded", "<i4"), ("_pad", "<i4")]
)
CFG_FIELDS = [
    ("surface_epsilon", "<f8", 1e-3),
    ("max_trace_steps", "<i8", 128),
    ("shadow_steps", "<i8", 256),
    ("ray_tmax", "<f8", 100.0),
    ("shadow_k", "<f8", 8.0),
    ("probe_visibility_k", "<f8", 8.0),
    ("gradient_step", "<f8", 1e-3),
    ("max_per_cluster", "<i8", 8),
    ("merge_radius", "<f8", 10.0),
    ("threshold1_frac", "<f8", 0.15),
    ("threshold2_frac", "<f8", 0.3),
    ("max_descent_steps", "<i8", 16),
    ("probe_budget", "<i8", 0),
    ("n_rays_full", "<i8", 144),
    ("hysteresis", "<f8", 0.9),
    ("alpha_min", "<f8", 0.02),
    ("bounce_coeff", "<f8", 0.9),
    ("oct_res", "<i8", 8),
    ("rotate_per_frame", "<i8", 1),
    ("seed", "<u8", 0),
    ("mvc_relocation_frac", "<f8", 0.25),
    ("dedup_quant_frac", "<f8", 0.25),
    ("contact_radius_frac", "<f8", 0.5),
    ("contact_samples", "<i8", 8),
    ("history_blend", "<f8", 0.6),
    ("depth_sigma_frac", "<f8", 0.1),
    ("exposure", "<f8", 1.0),
    ("fps", "<i8", 30),
]
CFG_DTYPE = np.dtype([(n, t) for n, t, _ in CFG_FIELDS])
PROBE_DTYPE = np.dtype(
    [
        ("resting", "<f8", (3,)),
        ("pos", "<f8", (3,)),
        ("last_pos", "<f8", (3,)),
        ("reject_history", "<i4"),
        ("alive", "<i4"),
        ("last_update_frame", "<i4"),
        ("_pad", "<i4"),
    ]
)
STATS_DTYPE = np.dtype(
    [
        ("sdf_queries", "<u8"),
        ("clusters_visited", "<u8"),
        ("clusters_skipped", "<u8"),
        ("primitive_evals", "<u8"),
        ("trace_steps", "<u8"),
        ("sphere_traces", "<u8"),
        ("shadow_traces", "<u8"),
        ("visibility_traces", "<u8"),
    ]
)
RAY_DTYPE = np.dtype(
    [
        ("dir", "<f8", (3,)),
        ("t", "<f8"),
        ("radiance", "<f8", (3,)),
        ("normal", "<f8", (3,)),
        ("converged", "<i4"),
        ("miss", "<i4"),
        ("prim_index", "<i4"),
        ("steps", "<i4"),
    ]
)
GBUFFER_DTYPE = np.dtype(
    [
        ("depth", "<f8"),
        ("normal", "<f8", (3,)),
        ("albedo", "<f8", (3,)),
        ("emission", "<f8", (3,)),
        ("world_pos", "<f8", (3,)),
        ("motion", "<f8", (2,)),
        ("prim_index", "<i4"),
        ("_pad", "<i4"),
    ]
)
CAMERA_DTYPE = np.dtype(
    [("position", "<f8", (3,)), ("forward", "<f8", (3,)), ("right", "<f8", (3,)), ("up", "<f8", (3,)),
     ("fov_y_deg", "<f8")]
)
assert GBUFFER_DTYPE.itemsize == 128 and CAMERA_DTYPE.itemsize == 104
assert PRIM_DTYPE.itemsize == 184 and LIGHT_DTYPE.itemsize == 80
assert CLUSTER_DTYPE.itemsize == 56 and CFG_DTYPE.itemsize == 224
assert PROBE_DTYPE.itemsize == 88 and RAY_DTYPE.itemsize == 96

SPHERE, BOX, PLANE, CYLINDER, CAPSULE = range(5)
LIGHT_POINT, LIGHT_DIRECTIONAL, LIGHT_SKY = range(3)

_HDR = struct.Struct("<4sI4I3d13d3iid")
assert _HDR.size == 176


def default_cfg(**overrides) -> np.ndarray:
    """RenderConfig defaults (config.hpp:9-50) as a 1-element sdfgi_cfg array."""
    cfg = np.zeros(1, CFG_DTYPE)
    for n, _, v in CFG_FIELDS:
        cfg[n] = v
    for k, v in overrides.items():
        if k not in CFG_DTYPE.names:
            raise KeyError(f"unknown config key {k}")
        cfg[k] = v
    return cfg


@dataclasses.dataclass
class Camera:
    position: np.ndarray
    forward: np.ndarray
    right: np.ndarray
    up: np.ndarray
    fov_y: float


@dataclasses.dataclass
class CascadeSpec:
    res: tuple
    spacing: float
    levels: int


@dataclasses.dataclass
class Scene:
    """Host-side image of ActiveScene (scene.hpp:88-103) plus the authoring context."""

    prims: np.ndarray  # PRIM_DTYPE
    lights: np.ndarray  # LIGHT_DTYPE
    clusters: np.ndarray  # CLUSTER_DTYPE
    member_start: np.ndarray  # int32[K+1]
    member_idx: np.ndarray  # int32[M]
    sky: np.ndarray  # float64[3]
    camera: Camera
    cascade: CascadeSpec
    cfg: np.ndarray  # CFG_DTYPE[1]

    @property
    def n_prims(self) -> int:
        return len(self.prims)

    @property
    def n_clusters(self) -> int:
        return len(self.clusters)


def read_sdfs(path) -> Scene:
    with open(path, "rb") as f:
        buf = f.read()
    h = _HDR.unpack_from(buf, 0)
    if h[0] != b"SDFS" or h[1] != 1:
        raise ValueError(f"{path}: not an SDFS v1 file")
    n_prims, n_lights, n_clusters, n_members = h[2:6]
    sky = np.array(h[6:9])
    cam = h[9:22]
    camera = Camera(
        np.array(cam[0:3]), np.array(cam[3:6]), np.array(cam[6:9]), np.array(cam[9:12]), cam[12]
    )
    res = tuple(h[22:25])
    cascade = CascadeSpec(res, h[26], h[25])
    off = _HDR.size
    cfg = np.frombuffer(buf, CFG_DTYPE, 1, off).copy()
    off += CFG_DTYPE.itemsize
    prims = np.frombuffer(buf, PRIM_DTYPE, n_prims, off).copy()
    off += PRIM_DTYPE.itemsize * n_prims
    lights = np.frombuffer(buf, LIGHT_DTYPE, n_lights, off).copy()
    off += LIGHT_DTYPE.itemsize * n_lights
    clusters = np.frombuffer(buf, CLUSTER_DTYPE, n_clusters, off).copy()
    off += CLUSTER_DTYPE.itemsize * n_clusters
    member_start = np.frombuffer(buf, "<i4", n_clusters + 1, off).copy()
    off += 4 * (n_clusters + 1)
    member_idx = np.frombuffer(buf, "<i4", n_members, off).copy()
    return Scene(prims, lights, clusters, member_start, member_idx, sky, camera, cascade, cfg)


def write_sdfs(path, s: Scene) -> None:
    hdr = _HDR.pack(
        b"SDFS",
        1,
        len(s.prims),
        len(s.lights),
        len(s.clusters),
        len(s.member_idx),
        *[float(x) for x in s.sky],
        *[float(x) for x in s.camera.position],
        *[float(x) for x in s.camera.forward],
        *[float(x) for x in s.camera.right],
        *[float(x) for x in s.camera.up],
        float(s.camera.fov_y),
        *[int(x) for x in s.cascade.res],
        int(s.cascade.levels),
        float(s.cascade.spacing),
    )
    parts = [
        hdr,
        np.ascontiguousarray(s.cfg, CFG_DTYPE).tobytes(),
        np.ascontiguousarray(s.prims, PRIM_DTYPE).tobytes(),
        np.ascontiguousarray(s.lights, LIGHT_DTYPE).tobytes(),
        np.ascontiguousarray(s.clusters, CLUSTER_DTYPE).tobytes(),
        np.ascontiguousarray(s.member_start, "<i4").tobytes(),
        np.ascontiguousarray(s.member_idx, "<i4").tobytes(),
    ]
    if (len(s.member_start) + len(s.member_idx)) % 2:
        parts.append(b"\0\0\0\0")
    with open(path, "wb") as f:
        f.write(b"".join(parts))


def read_sdfa(path):
    """ProbeAtlas::load (atlas.hpp:101-116): returns (res, probe_count, float32[P,R+2,R+2,3])."""
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:4] != b"SDFA":
        raise ValueError(f"{path}: not an SDFA file")
    _, r, n = struct.unpack_from("<3I", buf, 4)
    t = r + 2
    data = np.frombuffer(buf, "<f4", n * t * t * 3, 16).reshape(n, t, t, 3).copy()
    return r, n, data


def write_sdfa(path, atlas: np.ndarray) -> None:
    """ProbeAtlas::dump (atlas.hpp:89-99)."""
    n, t = atlas.shape[0], atlas.shape[1]
    with open(path, "wb") as f:
        f.write(b"SDFA" + struct.pack("<3I", 1, t - 2, n))
        f.write(np.ascontiguousarray(atlas, "<f4").tobytes())


# ------------------------------------------------------------- image.hpp:49-89
def write_sdfi(path, rgb, width, height) -> None:
    """writeHdr: "SDFI", u32 width, u32 height, u32 channels = 3, then row-major
    float32 triplets (each channel rounded from double as static_cast<float>)."""
    data = np.asarray(rgb, np.float64).reshape(-1)
    assert data.size == 3 * width * height
    with open(path, "wb") as f:
        f.write(b"SDFI")
        f.write(np.array([width, height, 3], "<u4").tobytes())
        f.write(data.astype("<f4").tobytes())


def read_sdfi(path):
    """readHdr -> (width, height, float32[h, w, 3])."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != b"SDFI":
        raise ValueError(f"bad SDFI file {path}")
    w, h, ch = np.frombuffer(raw[4:16], "<u4")
    if ch != 3:
        raise ValueError(f"SDFI channels {ch} != 3")
    img = np.frombuffer(raw[16:16 + 12 * int(w) * int(h)], "<f4").reshape(int(h), int(w), 3)
    return int(w), int(h), img.copy()


# -------------------------------------------------------- pipeline.hpp:11-42
METRICS_FIELDS = ["frame", "active_primitives", "clusters", "probes_total", "probes_updated", "relocated",
                  "rejected", "dead", "t_cull_ms", "t_probe_pos_ms", "t_probe_update_ms", "t_gbuffer_ms",
                  "t_visibility_ms", "t_gi_resolve_ms", "t_contact_ms", "t_compose_ms", "vis_traces_per_pixel",
                  "jitter_max_texel_delta"]


def metrics_csv_header() -> str:
    """FrameMetrics::csvHeader."""
    return ",".join(METRICS_FIELDS)


def _fmt_g(v, prec):
    """printf %.<prec>g (Python's 'g' matches C's for finite values)."""
    return f"{v:.{prec}g}"


def metrics_csv_row(m: dict) -> str:
    """FrameMetrics::csvRow: %d x8, %.3f x8, %.6f, %.6g."""
    ints = [str(int(m[k])) for k in METRICS_FIELDS[:8]]
    times = [f"{float(m[k]):.3f}" for k in METRICS_FIELDS[8:16]]
    return ",".join(ints + times + [f"{float(m['vis_traces_per_pixel']):.6f}",
                                    _fmt_g(float(m["jitter_max_texel_delta"]), 6)])
