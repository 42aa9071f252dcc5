"""Scene files, animation and per-frame scene instantiation —
the host side that turns an authored scene into the ActiveScene the device path
consumes, restated from the reference so a Python caller needs no reference code.

    parseScene / loadSceneFile   scene_file.hpp:205-450 (same grammar, checks and
                                 "line:col: message" SceneParseError)
    evalTrackVec / sceneAtTime   scene_file.hpp:560-650 (keyframe lerp; sky lights
                                 folded into the environment)
    primitiveAabb                primitives.hpp:112-151
    buildClusters                scene.hpp:110-178 (greedy surface-area agglomeration)
    cullAndLod                   scene.hpp:188-203 (distance LOD + re-clustering)
    buildCamera                  camera.hpp:15-26

All arithmetic is plain IEEE double in the reference's operation order (Python
floats have no FMA contraction and math.* is the same libm), so frame scenes are
bit-identical to the reference's (tests/test_scene_file.py, fixtures from the
reference itself). ``activeScene`` packs the result into the SDFS image
(scene_io.Scene) uploaded by ``Device.upload_scene``.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import scene_io as sio

INF = math.inf
CLUSTER_CULL_MARGIN = 1e-9  # kClusterCullMargin, scene.hpp:108


class SceneParseError(RuntimeError):
    """scene_file.hpp:65-74: message "line:col: what"."""

    def __init__(self, line, col, what):
        super().__init__(f"{line}:{col}: {what}")
        self.line, self.col = line, col


# ------------------------------------------------------------------ vec.hpp
def _add(a, b):
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _mul(a, s):
    return (a[0] * s, a[1] * s, a[2] * s)


def _div(a, s):
    return (a[0] / s, a[1] / s, a[2] / s)


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _length(a):
    return math.sqrt(_dot(a, a))


def _normalize(a):
    return _div(a, _length(a))


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _min(a, b):  # std::min
    return b if b < a else a


def _max(a, b):  # std::max
    return b if a < b else a


def _vmin(a, b):
    return (_min(a[0], b[0]), _min(a[1], b[1]), _min(a[2], b[2]))


def _vmax(a, b):
    return (_max(a[0], b[0]), _max(a[1], b[1]), _max(a[2], b[2]))


def _lerp(a, b, t):
    return _add(a, _mul(_sub(b, a), t))


IDENTITY = ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0))


def fromAxisAngle(axis, radians):
    """Mat3::fromAxisAngle, vec.hpp:80-94 (row-major)."""
    a = _normalize(axis)
    c, s = math.cos(radians), math.sin(radians)
    t = 1 - c
    return ((t * a[0] * a[0] + c, t * a[0] * a[1] - s * a[2], t * a[0] * a[2] + s * a[1]),
            (t * a[0] * a[1] + s * a[2], t * a[1] * a[1] + c, t * a[1] * a[2] - s * a[0]),
            (t * a[0] * a[2] - s * a[1], t * a[1] * a[2] + s * a[0], t * a[2] * a[2] + c))


def fromZTo(d):
    """Mat3::fromZTo, vec.hpp:97-104."""
    z = (0.0, 0.0, 1.0)
    c = _dot(z, d)
    if c > 1 - 1e-12:
        return IDENTITY
    if c < -1 + 1e-12:
        return fromAxisAngle((1.0, 0.0, 0.0), math.pi)
    return fromAxisAngle(_cross(z, d), math.acos(min(max(c, -1.0), 1.0)))


def _matvec(m, v):
    return (m[0][0] * v[0] + m[0][1] * v[1] + m[0][2] * v[2],
            m[1][0] * v[0] + m[1][1] * v[1] + m[1][2] * v[2],
            m[2][0] * v[0] + m[2][1] * v[1] + m[2][2] * v[2])


# ------------------------------------------------------------ scene_file.hpp
@dataclasses.dataclass
class PrimitiveSpec:
    kind: str = "sphere"
    position: tuple = (0.0, 0.0, 0.0)
    rotateAxis: tuple = (0.0, 0.0, 1.0)
    rotateDeg: float = 0.0
    size: list = dataclasses.field(default_factory=list)
    normal: tuple = (0.0, 0.0, 1.0)
    offset: float = 0.0
    hasNormal: bool = False
    albedo: tuple = (0.5, 0.5, 0.5)
    emission: tuple = (0.0, 0.0, 0.0)
    lodTier: int = 0
    id: int = -1


@dataclasses.dataclass
class LightSpec:
    kind: str = "point"
    position: tuple = (0.0, 0.0, 0.0)
    direction: tuple = (0.0, -1.0, 0.0)
    intensity: tuple = (1.0, 1.0, 1.0)


@dataclasses.dataclass
class Keyframe:
    time: float
    what: str  # "position" | "intensity"
    value: tuple


@dataclasses.dataclass
class Track:
    target: str = "primitive"  # "primitive" | "light"
    id: int = 0
    keys: list = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class CameraSpec:
    position: tuple = (0.0, 1.0, 5.0)
    lookAt: tuple = (0.0, 0.0, 0.0)
    up: tuple = (0.0, 1.0, 0.0)
    fovY: float = 60.0


@dataclasses.dataclass
class SceneFile:
    sky: tuple = (0.0, 0.0, 0.0)
    camera: CameraSpec = dataclasses.field(default_factory=CameraSpec)
    cascade: sio.CascadeSpec = dataclasses.field(default_factory=lambda: sio.CascadeSpec((6, 6, 6), 1.0, 1))
    config: np.ndarray = dataclasses.field(default_factory=sio.default_cfg)
    lodDistances: list = dataclasses.field(default_factory=list)
    primitives: list = dataclasses.field(default_factory=list)
    lights: list = dataclasses.field(default_factory=list)
    tracks: list = dataclasses.field(default_factory=list)


def _tokenize(text):
    """detail::tokenize, scene_file.hpp:80-116: words and braces with line:col."""
    out, line, col, i, n = [], 1, 1, 0, len(text)
    while i < n:
        c = text[i]
        if c == "#":
            while i < n and text[i] != "\n":
                i += 1
            continue
        if c == "\n":
            line += 1
            col = 1
            i += 1
            continue
        if c in " \t\r":
            col += 1
            i += 1
            continue
        if c in "{}":
            out.append((c, line, col))
            col += 1
            i += 1
            continue
        start, sc = i, col
        while i < n and not text[i].isspace() and text[i] not in "{}#":
            i += 1
            col += 1
        out.append((text[start:i], line, sc))
    return out


def _number(s):
    """strtod over the whole token (None if it is not one)."""
    try:
        v = float(s)
    except ValueError:
        return None
    return v if s.strip() == s else None


class _Cursor:
    """detail::Cursor, scene_file.hpp:118-200."""

    def __init__(self, toks):
        self.toks, self.pos = toks, 0

    def done(self):
        return self.pos >= len(self.toks)

    def peek(self):
        return self.toks[self.pos]

    def next(self):
        t = self.toks[self.pos]
        self.pos += 1
        return t

    def fail(self, at, msg):
        raise SceneParseError(at[1], at[2], msg)

    def _last(self):
        return (self.toks[-1][1], self.toks[-1][2]) if self.toks else (1, 1)

    def expectWord(self, what):
        if self.done():
            raise SceneParseError(*self._last(), f"expected {what}")
        t = self.next()
        if t[0] in ("{", "}"):
            self.fail(t, f"expected {what}")
        return t

    def expectNumber(self, what):
        t = self.expectWord(what)
        v = _number(t[0])
        if v is None:
            self.fail(t, f"expected a number for {what}, got '{t[0]}'")
        return v

    def expectInt(self, what):
        t = self.expectWord(what)
        try:
            v = int(t[0], 10)
        except ValueError:
            self.fail(t, f"expected an integer for {what}, got '{t[0]}'")
        return v

    def expectVec3(self, what):
        return (self.expectNumber(what), self.expectNumber(what), self.expectNumber(what))

    def expectOpen(self, key):
        if self.done() or self.peek()[0] != "{":
            self.fail(key, "expected '{' after block name")
        self.next()

    def atClose(self):
        return not self.done() and self.peek()[0] == "}"

    def expectClose(self, key):
        if self.done():
            self.fail(key, "unterminated block (missing '}')")
        self.next()


_CFG_KEYS = {  # config block key -> (cfg field, int?)
    "surface_epsilon": ("surface_epsilon", False), "max_trace_steps": ("max_trace_steps", True),
    "shadow_steps": ("shadow_steps", True), "ray_tmax": ("ray_tmax", False), "shadow_k": ("shadow_k", False),
    "probe_visibility_k": ("probe_visibility_k", False), "gradient_step": ("gradient_step", False),
    "max_per_cluster": ("max_per_cluster", True), "merge_radius": ("merge_radius", False),
    "threshold1_frac": ("threshold1_frac", False), "threshold2_frac": ("threshold2_frac", False),
    "max_descent_steps": ("max_descent_steps", True), "probe_budget": ("probe_budget", True),
    "n_rays": ("n_rays_full", True), "hysteresis": ("hysteresis", False), "alpha_min": ("alpha_min", False),
    "bounce_coeff": ("bounce_coeff", False), "oct_res": ("oct_res", True),
    "rotate_per_frame": ("rotate_per_frame", True), "seed": ("seed", True),
    "mvc_relocation_frac": ("mvc_relocation_frac", False), "dedup_quant_frac": ("dedup_quant_frac", False),
    "contact_radius_frac": ("contact_radius_frac", False), "contact_samples": ("contact_samples", True),
    "history_blend": ("history_blend", False), "depth_sigma_frac": ("depth_sigma_frac", False),
    "exposure": ("exposure", False), "fps": ("fps", True),
}


def _nonneg(cur, at, v, field):
    if not all(x >= 0 and math.isfinite(x) for x in v):
        cur.fail(at, f"{field} must be finite and >= 0")


def _color01(cur, at, v, field):
    if not all(0 <= x <= 1 for x in v):
        cur.fail(at, f"{field} must be in [0,1]")


def parseScene(text: str) -> SceneFile:
    """parseScene, scene_file.hpp:205-450."""
    cur = _Cursor(_tokenize(text))
    scene = SceneFile()
    autoId = 0
    while not cur.done():
        key = cur.next()
        k0 = key[0]
        if k0 == "sky":
            scene.sky = cur.expectVec3("sky")
            _nonneg(cur, key, scene.sky, "sky")
        elif k0 == "lod_distances":
            scene.lodDistances = []
            while not cur.done() and cur.peek()[0] not in ("{", "}") and _number(cur.peek()[0]) is not None:
                scene.lodDistances.append(cur.expectNumber("lod_distances"))
            for i in range(1, len(scene.lodDistances)):
                if scene.lodDistances[i] <= scene.lodDistances[i - 1]:
                    cur.fail(key, "lod_distances must be ascending")
        elif k0 == "camera":
            cur.expectOpen(key)
            cam = scene.camera
            while not cur.atClose():
                k = cur.expectWord("camera key")
                if k[0] == "position":
                    cam.position = cur.expectVec3("position")
                elif k[0] == "look_at":
                    cam.lookAt = cur.expectVec3("look_at")
                elif k[0] == "up":
                    cam.up = cur.expectVec3("up")
                elif k[0] == "fov_y":
                    cam.fovY = cur.expectNumber("fov_y")
                else:
                    cur.fail(k, f"unknown key '{k[0]}' in camera block")
            cur.expectClose(key)
            if not (0 < cam.fovY < 180):
                cur.fail(key, "fov_y must be in (0, 180)")
        elif k0 == "cascade":
            cur.expectOpen(key)
            res, sp, lv = list(scene.cascade.res), scene.cascade.spacing, scene.cascade.levels
            while not cur.atClose():
                k = cur.expectWord("cascade key")
                if k[0] == "resolution":
                    res = [cur.expectInt("resolution") for _ in range(3)]
                    if min(res) < 2:
                        cur.fail(k, "cascade resolution must be at least 2 per axis")
                elif k[0] == "spacing":
                    sp = cur.expectNumber("spacing")
                    if not sp > 0:
                        cur.fail(k, "spacing must be positive")
                elif k[0] == "levels":
                    lv = cur.expectInt("levels")
                    if lv < 1:
                        cur.fail(k, "levels must be >= 1")
                else:
                    cur.fail(k, f"unknown key '{k[0]}' in cascade block")
            cur.expectClose(key)
            scene.cascade = sio.CascadeSpec(tuple(res), sp, lv)
        elif k0 == "config":
            cur.expectOpen(key)
            c = scene.config
            while not cur.atClose():
                k = cur.expectWord("config key")
                if k[0] not in _CFG_KEYS:
                    cur.fail(k, f"unknown key '{k[0]}' in config block")
                field, isint = _CFG_KEYS[k[0]]
                v = cur.expectInt(k[0]) if isint else cur.expectNumber(k[0])
                if field == "rotate_per_frame":
                    v = 1 if v != 0 else 0
                c[field] = v
            cur.expectClose(key)
            if not (0 <= c["hysteresis"][0] < 1):
                cur.fail(key, "hysteresis must be in [0,1)")
            if not (0 <= c["bounce_coeff"][0] <= 1):
                cur.fail(key, "bounce_coeff must be in [0,1]")
            if c["n_rays_full"][0] < 8:
                cur.fail(key, "n_rays must be >= 8")
        elif k0 == "primitive":
            cur.expectOpen(key)
            p = PrimitiveSpec()
            kindTok = key
            while not cur.atClose():
                k = cur.expectWord("primitive key")
                if k[0] == "kind":
                    kindTok = cur.expectWord("kind")
                    p.kind = kindTok[0]
                    if p.kind not in ("sphere", "box", "plane", "cylinder", "capsule"):
                        cur.fail(kindTok, f"unknown primitive kind '{p.kind}'")
                elif k[0] == "position":
                    p.position = cur.expectVec3("position")
                elif k[0] == "rotate":
                    p.rotateAxis = cur.expectVec3("rotate axis")
                    p.rotateDeg = cur.expectNumber("rotate angle")
                    if _length(p.rotateAxis) < 1e-9:
                        cur.fail(k, "rotate axis must be nonzero")
                elif k[0] == "size":
                    p.size = []
                    while not cur.done() and cur.peek()[0] not in ("{", "}") and _number(cur.peek()[0]) is not None:
                        v = cur.expectNumber("size")
                        if not v > 0:
                            cur.fail(k, "size values must be strictly positive")
                        p.size.append(v)
                elif k[0] == "normal":
                    p.normal = cur.expectVec3("normal")
                    p.hasNormal = True
                    if _length(p.normal) < 1e-9:
                        cur.fail(k, "plane normal must be nonzero")
                elif k[0] == "offset":
                    p.offset = cur.expectNumber("offset")
                elif k[0] == "albedo":
                    p.albedo = cur.expectVec3("albedo")
                    _color01(cur, k, p.albedo, "albedo")
                elif k[0] == "emission":
                    p.emission = cur.expectVec3("emission")
                    _nonneg(cur, k, p.emission, "emission")
                elif k[0] == "lod_tier":
                    p.lodTier = cur.expectInt("lod_tier")
                    if p.lodTier < 0:
                        cur.fail(k, "lod_tier must be >= 0")
                elif k[0] == "id":
                    p.id = cur.expectInt("id")
                else:
                    cur.fail(k, f"unknown key '{k[0]}' in primitive block")
            cur.expectClose(key)
            want = {"sphere": 1, "box": 3, "plane": 0}.get(p.kind, 2)
            if len(p.size) != want:
                cur.fail(kindTok, f"primitive kind '{p.kind}' needs {want} size value(s), got {len(p.size)}")
            if p.id < 0:
                p.id = autoId
            autoId += 1
            if any(o.id == p.id for o in scene.primitives):
                cur.fail(key, f"duplicate primitive id {p.id}")
            scene.primitives.append(p)
        elif k0 == "light":
            cur.expectOpen(key)
            lt = LightSpec()
            while not cur.atClose():
                k = cur.expectWord("light key")
                if k[0] == "kind":
                    kt = cur.expectWord("kind")
                    lt.kind = kt[0]
                    if lt.kind not in ("point", "directional", "sky"):
                        cur.fail(kt, f"unknown light kind '{lt.kind}'")
                elif k[0] == "position":
                    lt.position = cur.expectVec3("position")
                elif k[0] == "direction":
                    lt.direction = cur.expectVec3("direction")
                    if _length(lt.direction) < 1e-9:
                        cur.fail(k, "direction must be nonzero")
                elif k[0] == "intensity":
                    lt.intensity = cur.expectVec3("intensity")
                    _nonneg(cur, k, lt.intensity, "intensity")
                else:
                    cur.fail(k, f"unknown key '{k[0]}' in light block")
            cur.expectClose(key)
            scene.lights.append(lt)
        elif k0 == "animate":
            cur.expectOpen(key)
            t = Track()
            sawTarget = False
            while not cur.atClose():
                k = cur.expectWord("animate key")
                if k[0] == "target":
                    what = cur.expectWord("target kind")
                    if what[0] not in ("primitive", "light"):
                        cur.fail(what, "animate target must be 'primitive' or 'light'")
                    t.target = what[0]
                    t.id = cur.expectInt("target id")
                    sawTarget = True
                elif k[0] == "key":
                    tm = cur.expectNumber("key time")
                    what = cur.expectWord("key property")
                    if what[0] not in ("position", "intensity"):
                        cur.fail(what, "key property must be 'position' or 'intensity'")
                    val = cur.expectVec3("key value")
                    if t.keys and tm <= t.keys[-1].time:
                        cur.fail(k, "keyframe times must be strictly increasing")
                    t.keys.append(Keyframe(tm, what[0], val))
                else:
                    cur.fail(k, f"unknown key '{k[0]}' in animate block")
            cur.expectClose(key)
            if not sawTarget:
                cur.fail(key, "animate block needs a target")
            if not t.keys:
                cur.fail(key, "animate block needs at least one key")
            scene.tracks.append(t)
        else:
            cur.fail(key, f"unknown top-level key '{k0}'")
    for t in scene.tracks:
        if t.target == "primitive":
            if not any(p.id == t.id for p in scene.primitives):
                raise SceneParseError(1, 1, f"animate target primitive id {t.id} does not exist")
        elif not 0 <= t.id < len(scene.lights):
            raise SceneParseError(1, 1, f"animate target light index {t.id} does not exist")
    return scene


def loadSceneFile(path: str) -> SceneFile:
    with open(path, "rb") as f:
        return parseScene(f.read().decode("latin-1"))


def evalTrackVec(keys, what, time, fallback):
    """scene_file.hpp:560-574: hold before the first key and after the last, lerp between."""
    prev = None
    for k in keys:
        if k.what != what:
            continue
        if k.time >= time:
            if prev is None:
                return k.value
            span = k.time - prev.time
            t = (time - prev.time) / span if span > 0 else 0
            return _lerp(prev.value, k.value, t)
        prev = k
    return prev.value if prev is not None else fallback


@dataclasses.dataclass
class Primitive:
    """SdfPrimitive (primitives.hpp:11-38)."""

    id: int
    kind: int
    rot: tuple
    trans: tuple
    size: tuple
    albedo: tuple
    emission: tuple
    lodTier: int


@dataclasses.dataclass
class SceneState:
    primitives: list
    lights: np.ndarray  # LIGHT_DTYPE
    sky: tuple


_KINDS = {"sphere": sio.SPHERE, "box": sio.BOX, "plane": sio.PLANE, "cylinder": sio.CYLINDER, "capsule": sio.CAPSULE}


def sceneAtTime(s: SceneFile, time: float) -> SceneState:
    """scene_file.hpp:584-645."""
    prims = []
    for spec in s.primitives:
        kind = _KINDS[spec.kind]
        if spec.kind == "sphere":
            size = (spec.size[0], 0.0, 0.0)
        elif spec.kind == "box":
            size = (spec.size[0], spec.size[1], spec.size[2])
        elif spec.kind == "plane":
            size = (1.0, 1.0, 1.0)  # SdfPrimitive::size default (primitives.hpp:35), unused by a plane
        else:
            size = (spec.size[0], spec.size[1], 0.0)
        pos = spec.position
        for t in s.tracks:
            if t.target == "primitive" and t.id == spec.id:
                pos = evalTrackVec(t.keys, "position", time, pos)
        rot = IDENTITY
        if spec.kind == "plane" and spec.hasNormal:
            n = _normalize(spec.normal)
            rot = fromZTo(n)
            trans = _add(_mul(n, spec.offset), pos)
        else:
            if spec.rotateDeg != 0:
                rot = fromAxisAngle(spec.rotateAxis, spec.rotateDeg * math.pi / 180.0)
            trans = pos
        prims.append(Primitive(spec.id, kind, rot, trans, size, spec.albedo, spec.emission, spec.lodTier))
    sky = s.sky
    lights = []
    for i, spec in enumerate(s.lights):
        intensity, pos = spec.intensity, spec.position
        for t in s.tracks:
            if t.target != "light" or t.id != i:
                continue
            intensity = evalTrackVec(t.keys, "intensity", time, intensity)
            pos = evalTrackVec(t.keys, "position", time, pos)
        if spec.kind == "sky":
            sky = _add(sky, intensity)
            continue
        rec = np.zeros(1, sio.LIGHT_DTYPE)
        rec["kind"] = sio.LIGHT_POINT if spec.kind == "point" else sio.LIGHT_DIRECTIONAL
        rec["position"] = pos
        rec["direction"] = _normalize(spec.direction)
        rec["intensity"] = intensity
        lights.append(rec)
    lt = np.concatenate(lights) if lights else np.zeros(0, sio.LIGHT_DTYPE)
    return SceneState(prims, lt, sky)


def primitiveAabb(p: Primitive):
    """primitives.hpp:112-151 -> (lo, hi)."""
    lo, hi = (INF, INF, INF), (-INF, -INF, -INF)

    def expand(q):
        nonlocal lo, hi
        lo, hi = _vmin(lo, q), _vmax(hi, q)

    r, t = p.rot, p.trans

    def local_box(h):
        e = tuple(abs(r[i][0]) * h[0] + abs(r[i][1]) * h[1] + abs(r[i][2]) * h[2] for i in range(3))
        expand(_sub(t, e))
        expand(_add(t, e))

    if p.kind == sio.SPHERE:
        s = p.size[0]
        expand(_sub(t, (s, s, s)))
        expand(_add(t, (s, s, s)))
    elif p.kind == sio.BOX:
        local_box(p.size)
    elif p.kind == sio.PLANE:
        expand((-1e9, -1e9, -1e9))
        expand((1e9, 1e9, 1e9))
    elif p.kind == sio.CYLINDER:
        local_box((p.size[0], p.size[0], p.size[1]))
    else:
        a = _add(_matvec(r, (0.0, 0.0, -p.size[1])), t)
        b = _add(_matvec(r, (0.0, 0.0, p.size[1])), t)
        s = p.size[0]
        expand(_sub(_vmin(a, b), (s, s, s)))
        expand(_add(_vmax(a, b), (s, s, s)))
    return lo, hi


def _area(lo, hi):
    if not lo[0] <= hi[0]:
        return 0
    e = _sub(hi, lo)
    return 2 * (e[0] * e[1] + e[1] * e[2] + e[2] * e[0])


def buildClusters(prims, maxPerCluster, mergeRadius):
    """scene.hpp:110-178: greedy agglomeration of the admissible pair whose merged box
    grows the total surface area least. Returns [(cullLo, cullHi, members, unbounded)]."""
    work = []
    for i, p in enumerate(prims):
        lo, hi = primitiveAabb(p)
        unb = p.kind == sio.PLANE
        c = p.trans if unb else _mul(_add(lo, hi), 0.5)
        work.append({"lo": lo, "hi": hi, "c": c, "m": [i], "unb": unb, "alive": True})
    while True:
        bestA = bestB = -1
        bestCost = INF
        n = len(work)
        for a in range(n):
            wa = work[a]
            if not wa["alive"] or wa["unb"]:
                continue
            for b in range(a + 1, n):
                wb = work[b]
                if not wb["alive"] or wb["unb"]:
                    continue
                if len(wa["m"]) + len(wb["m"]) > maxPerCluster:
                    continue
                if _length(_sub(wa["c"], wb["c"])) > mergeRadius:
                    continue
                ulo, uhi = _vmin(wa["lo"], wb["lo"]), _vmax(wa["hi"], wb["hi"])
                cost = _area(ulo, uhi) - _area(wa["lo"], wa["hi"]) - _area(wb["lo"], wb["hi"])
                if cost < bestCost:
                    bestCost, bestA, bestB = cost, a, b
        if bestA < 0:
            break
        wa, wb = work[bestA], work[bestB]
        wa["lo"], wa["hi"] = _vmin(wa["lo"], wb["lo"]), _vmax(wa["hi"], wb["hi"])
        wa["m"] = wa["m"] + wb["m"]
        wa["c"] = _mul(_add(wa["lo"], wa["hi"]), 0.5)
        wb["alive"] = False
    m = CLUSTER_CULL_MARGIN
    return [(_sub(w["lo"], (m, m, m)), _add(w["hi"], (m, m, m)), w["m"], w["unb"]) for w in work if w["alive"]]


def _boxDistance(lo, hi, p):
    d = _vmax(_vmax(_sub(lo, p), _sub(p, hi)), (0.0, 0.0, 0.0))
    return _length(d)


def cullAndLod(prims, cameraPos, lodDistances, maxPerCluster=8, mergeRadius=10.0):
    """scene.hpp:188-203: tier >= 1 primitives farther than their tier's distance are
    dropped; clusters are rebuilt over the survivors. Returns (prims, clusters)."""
    keep = []
    for p in prims:
        if p.lodTier >= 1 and lodDistances:
            idx = min(p.lodTier - 1, len(lodDistances) - 1)
            lo, hi = primitiveAabb(p)
            if _boxDistance(lo, hi, tuple(cameraPos)) > lodDistances[idx]:
                continue
        keep.append(p)
    clusters = buildClusters(keep, maxPerCluster, mergeRadius) if keep else []
    return keep, clusters


def buildCamera(spec: CameraSpec) -> sio.Camera:
    """Camera::lookAt, camera.hpp:15-26."""
    pos = spec.position
    f = _normalize(_sub(spec.lookAt, pos))
    r = _cross(f, spec.up)
    if _length(r) < 1e-9:
        r = _cross(f, (1.0, 0.0, 0.0))
    r = _normalize(r)
    u = _cross(r, f)
    return sio.Camera(np.array(pos), np.array(f), np.array(r), np.array(u), float(spec.fovY))


def packScene(prims, clusters, lights, sky, camera, cascade, cfg) -> sio.Scene:
    """An ActiveScene (primitives + buildClusters output) as an SDFS image."""
    pr = np.zeros(len(prims), sio.PRIM_DTYPE)
    for i, p in enumerate(prims):
        pr[i]["id"], pr[i]["kind"], pr[i]["lod_tier"] = p.id, p.kind, p.lodTier
        pr[i]["rot"] = [p.rot[a][b] for a in range(3) for b in range(3)]
        pr[i]["trans"], pr[i]["size"] = p.trans, p.size
        pr[i]["albedo"], pr[i]["emission"] = p.albedo, p.emission
    cl = np.zeros(len(clusters), sio.CLUSTER_DTYPE)
    start, idx = [0], []
    for k, (lo, hi, members, unb) in enumerate(clusters):
        cl[k]["lo"], cl[k]["hi"], cl[k]["unbounded"] = lo, hi, 1 if unb else 0
        idx.extend(members)
        start.append(len(idx))
    return sio.Scene(pr, lights, cl, np.array(start, np.int32), np.array(idx, np.int32),
                     np.array(sky, np.float64), camera, cascade, np.array(cfg, sio.CFG_DTYPE).reshape(1).copy())


def activeScene(s: SceneFile, time: float, cameraPos=None) -> sio.Scene:
    """The frame's ActiveScene as an SDFS image: sceneAtTime + cullAndLod
    (pipeline.hpp:95-103) with the scene's clustering parameters."""
    cam = buildCamera(s.camera)
    state = sceneAtTime(s, time)
    cp = cam.position if cameraPos is None else cameraPos
    prims, clusters = cullAndLod(state.primitives, cp, s.lodDistances, int(s.config["max_per_cluster"][0]),
                                 float(s.config["merge_radius"][0]))
    return packScene(prims, clusters, state.lights, state.sky, cam, s.cascade, s.config)
