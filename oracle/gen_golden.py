#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

TEST INFRASTRUCTURE. Runs oracle/_ref/ref_parity (the unmodified reference headers
under /root/reference compiled with -ffp-contract=off by oracle/Makefile) and
packs its dumps into tests/golden/<case>/{scene.sdfs, summary.json, data.npz}.
Only this container can regenerate them (the GPU box has no /root/reference);
the fixtures are committed.

Cases:
  c1        Cornell, 8x8x8 probes spacing 1, 64 rays, 3 passes (frames 0,1,2)
  sponza    sponza-lite at its own 12x7x9 grid, 32 rays, 2 passes (cylinders,
            directional + point light, sky, relocation, MVC bounce)
  thinwall  two-room-thin-wall, 32 rays, 2 passes (thin occluder)
  openfield open-field-cascade: 3 cascades, ground plane (unbounded cluster), 16 rays
  furnace   4x4x4 emissive enclosure, 256 rays, 1 pass (bounce 0)
  kinds     synthetic: every primitive kind, rotated, reference-built clusters, 24 rays
"""
from __future__ import annotations

import json
import math
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2007_14394_b200 import scene_io  # noqa: E402

REF = os.path.join(HERE, "_ref", "ref_parity")
SCENES = "/root/reference/proj/scenes"
OUT = os.path.join(ROOT, "tests", "golden")


def run(*args):
    r = subprocess.run([REF, *map(str, args)], check=True, capture_output=True, text=True)
    return r.stdout


def axis_angle(axis, deg):
    a = np.asarray(axis, float)
    a = a / np.linalg.norm(a)
    th = math.radians(deg)
    c, s, t = math.cos(th), math.sin(th), 1 - math.cos(th)
    x, y, z = a
    return np.array(
        [
            [t * x * x + c, t * x * y - s * z, t * x * z + s * y],
            [t * x * y + s * z, t * y * y + c, t * y * z - s * x],
            [t * x * z - s * y, t * y * z + s * x, t * z * z + c],
        ]
    )


def kinds_scene(path):
    """Small synthetic scene with every PrimitiveKind (primitives.hpp:9), rotations,
    an unbounded plane, emissive members, a point and a directional light."""
    rng = np.random.default_rng(7)
    prims = []
    pid = 0

    def add(kind, pos, size, rot=None, albedo=(0.6, 0.6, 0.6), emission=(0, 0, 0)):
        nonlocal pid
        p = np.zeros(1, scene_io.PRIM_DTYPE)
        p["id"] = pid
        pid += 1
        p["kind"] = kind
        p["rot"] = (np.eye(3) if rot is None else rot).reshape(9)
        p["trans"] = pos
        p["size"] = size
        p["albedo"] = albedo
        p["emission"] = emission
        prims.append(p)

    add(scene_io.PLANE, (0, 0, 0), (0, 0, 0), axis_angle((1, 0, 0), -90), albedo=(0.5, 0.45, 0.4))
    for i in range(22):
        kind = [scene_io.SPHERE, scene_io.BOX, scene_io.CYLINDER, scene_io.CAPSULE][i % 4]
        pos = (rng.uniform(-3, 3), rng.uniform(0.2, 2.5), rng.uniform(-3, 3))
        r = rng.uniform(0.15, 0.5)
        if kind == scene_io.SPHERE:
            size = (r, 0, 0)
        elif kind == scene_io.BOX:
            size = (r, rng.uniform(0.1, 0.6), rng.uniform(0.1, 0.6))
        else:
            size = (r, rng.uniform(0.2, 0.7), 0)
        rot = axis_angle(rng.normal(size=3), rng.uniform(0, 180)) if i % 3 else None
        em = (1.5, 1.2, 0.8) if i == 5 else (0, 0, 0)
        add(kind, pos, size, rot, tuple(rng.uniform(0.2, 0.8, 3)), em)
    prims = np.concatenate(prims)
    lights = np.zeros(2, scene_io.LIGHT_DTYPE)
    lights[0]["kind"] = scene_io.LIGHT_POINT
    lights[0]["position"] = (0.5, 3.5, 0.2)
    lights[0]["intensity"] = (9, 9, 8)
    lights[1]["kind"] = scene_io.LIGHT_DIRECTIONAL
    d = np.array([0.3, -1.0, 0.2])
    lights[1]["direction"] = d / np.linalg.norm(d)
    lights[1]["intensity"] = (1.2, 1.1, 1.0)
    cam = scene_io.Camera(
        np.array([0.0, 1.5, 0.0]), np.array([0, 0, -1.0]), np.array([1.0, 0, 0]),
        np.array([0, 1.0, 0]), 60.0,
    )
    s = scene_io.Scene(
        prims, lights, np.zeros(0, scene_io.CLUSTER_DTYPE), np.zeros(1, np.int32),
        np.zeros(0, np.int32), np.array([0.2, 0.25, 0.3]), cam,
        scene_io.CascadeSpec((8, 4, 8), 0.9, 1), scene_io.default_cfg(),
    )
    tmp = path + ".noclusters"
    scene_io.write_sdfs(tmp, s)
    run("recluster", tmp, path, 4, 3.0)
    os.remove(tmp)


CASES = {
    "c1": dict(scene="cornell.scene", passes=3, extra=["--res", 8, 8, 8, "--spacing", 1.0,
                                                        "--nrays", 64], debug=[0, 9, 100, 300, 455]),
    "sponza": dict(scene="sponza-lite.scene", passes=2, extra=["--nrays", 32], debug=[5, 200, 431]),
    "thinwall": dict(scene="two-room-thin-wall.scene", passes=2, extra=["--nrays", 32], debug=[77, 250]),
    "openfield": dict(scene="open-field-cascade.scene", passes=2, extra=["--nrays", 16], debug=[40]),
    "furnace": dict(scene="furnace.scene", passes=1, extra=[], debug=[21]),
    "kinds": dict(scene=None, passes=2, extra=["--nrays", 24], debug=[3, 70, 200]),
    # budgeted scheduling (selectProbesForUpdate, probe_volume.hpp:154-198): forced
    # staleness kicks in after ceil(total / budget) frames
    "sched_c1": dict(scene="cornell.scene", passes=8, extra=["--res", 8, 8, 8, "--spacing", 1.0, "--nrays", 32,
                                                              "--budget", 96], debug=[]),
    "sched_openfield": dict(scene="open-field-cascade.scene", passes=6, extra=["--nrays", 8, "--budget", 200],
                            debug=[]),
}


def build_case(name, spec):
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    sdfs = os.path.join(d, "scene.sdfs")
    if spec["scene"]:
        run("scene", os.path.join(SCENES, spec["scene"]), sdfs)
    else:
        kinds_scene(sdfs)
    with tempfile.TemporaryDirectory() as tmp:
        args = ["passes", sdfs, tmp, "--passes", spec["passes"], "--threads", 2, *spec["extra"]]
        for p in spec["debug"]:
            args += ["--debug-probe", p]
        summary = json.loads(run(*args))
        data = {}
        for fn in sorted(os.listdir(tmp)):
            base, ext = os.path.splitext(fn)
            path = os.path.join(tmp, fn)
            if ext == ".sdfa":
                data[base] = scene_io.read_sdfa(path)[2]
            elif base.startswith("probes"):
                data[base] = np.fromfile(path, scene_io.PROBE_DTYPE)
            elif base.startswith("rays"):
                data[base] = np.fromfile(path, scene_io.RAY_DTYPE)
            elif base.startswith("refs"):
                data[base] = np.fromfile(path, "<i4").reshape(-1, 2)
    summary["case"] = name
    summary["args"] = [str(a) for a in args[3:]]
    summary["debug_probes"] = spec["debug"]
    summary["generator"] = "oracle/gen_golden.py via oracle/_ref/ref_parity (-ffp-contract=off)"
    with open(os.path.join(d, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    np.savez_compressed(os.path.join(d, "data.npz"), **data)
    print(name, {k: v.shape for k, v in data.items()})


# C3 gather fixtures: probe passes, then renderGBuffer + the gather stages for two
# frames (frame 0 without history, frame 1 with) at a small resolution.
GATHER_CASES = {
    "gather_c1": dict(src="c1", passes=2, extra=["--res", 8, 8, 8, "--spacing", 1.0, "--nrays", 64], size=(96, 64)),
    "gather_sponza": dict(src="sponza", passes=2, extra=["--nrays", 32], size=(128, 72)),
    "gather_openfield": dict(src="openfield", passes=1, extra=["--nrays", 16], size=(96, 54)),
}


# C5 dynamic sequences: sceneAtTime + cullAndLod per frame, the probe pass on
# persistent cascades; every frame's active scene, probes/atlas every `every` frames.
DYNAMIC_CASES = {
    "dyn_sphere": dict(scene=os.path.join(SCENES, "dynamic-sphere.scene"), frames=60, every=12,
                       extra=["--nrays", 32]),
    "dyn_light": dict(scene=os.path.join(HERE, "scenes", "dynamic-light.scene"), frames=40, every=13,
                      extra=["--nrays", 24]),
}


# The reference's whole frame loop (Renderer::renderFrame): composed images + metrics.
RENDER_CASES = {
    "render_dynsphere": dict(scene=os.path.join(SCENES, "dynamic-sphere.scene"), frames=12, size=(80, 48),
                             extra=["--nrays", 32]),
    "render_light": dict(scene=os.path.join(HERE, "scenes", "dynamic-light.scene"), frames=8, size=(64, 40),
                         extra=["--nrays", 24]),
}


def build_render_case(name, spec):
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        args = ["render", spec["scene"], tmp, "--passes", spec["frames"], "--threads", 2, "--size", *spec["size"],
                *spec["extra"]]
        summary = json.loads(run(*args))
        data = {}
        for fn in sorted(os.listdir(tmp)):
            base, ext = os.path.splitext(fn)
            path = os.path.join(tmp, fn)
            if ext == ".sdfi":
                data[base] = scene_io.read_sdfi(path)[2]
                if base == "image_f0":
                    data["image_f0_bytes"] = np.fromfile(path, np.uint8)
        with open(os.path.join(tmp, "metrics.csv")) as f:
            summary["metrics_csv"] = f.read()
    with open(spec["scene"]) as f:
        summary["scene_text"] = f.read()
    summary.update(case=name, args=[str(a) for a in args[3:]], size=list(spec["size"]),
                   generator="oracle/gen_golden.py via oracle/_ref/ref_parity render (Renderer::renderFrame)")
    with open(os.path.join(d, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    np.savez_compressed(os.path.join(d, "data.npz"), **data)
    print(name, len(data), "arrays")


def build_dynamic_case(name, spec):
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        args = ["dynamic", spec["scene"], tmp, "--passes", spec["frames"], "--threads", 2, "--dump-every",
                spec["every"], *spec["extra"]]
        summary = json.loads(run(*args))
        data = {}
        for fn in sorted(os.listdir(tmp)):
            base, ext = os.path.splitext(fn)
            path = os.path.join(tmp, fn)
            if ext == ".sdfa":
                data[base] = scene_io.read_sdfa(path)[2]
            elif base.startswith("probes"):
                data[base] = np.fromfile(path, scene_io.PROBE_DTYPE)
            elif ext == ".sdfs":
                sc = scene_io.read_sdfs(path)
                f = base.split("_")[-1]
                data[f"prims_{f}"] = sc.prims
                data[f"lights_{f}"] = sc.lights
                data[f"clusters_{f}"] = sc.clusters
                data[f"mstart_{f}"] = sc.member_start
                data[f"midx_{f}"] = sc.member_idx
                data[f"sky_{f}"] = sc.sky
    with open(spec["scene"]) as f:
        scene_text = f.read()
    summary.update(case=name, args=[str(a) for a in args[3:]], frames_total=spec["frames"], every=spec["every"],
                   scene_text=scene_text,
                   generator="oracle/gen_golden.py via oracle/_ref/ref_parity dynamic (-ffp-contract=off)")
    with open(os.path.join(d, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    np.savez_compressed(os.path.join(d, "data.npz"), **data)
    print(name, len(data), "arrays")


def build_gather_case(name, spec):
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    sdfs = os.path.join(OUT, spec["src"], "scene.sdfs")
    with tempfile.TemporaryDirectory() as tmp:
        args = ["gather", sdfs, tmp, "--passes", spec["passes"], "--threads", 2, *spec["extra"],
                "--size", *spec["size"], "--gather-frames", 2]
        summary = json.loads(run(*args))
        data = {}
        for fn in sorted(os.listdir(tmp)):
            base, ext = os.path.splitext(fn)
            path = os.path.join(tmp, fn)
            if ext == ".sdfa":
                data[base] = scene_io.read_sdfa(path)[2]
            elif base == "gbuffer":
                data[base] = np.fromfile(path, scene_io.GBUFFER_DTYPE)
            elif base.startswith("gprobes"):
                data[base] = np.fromfile(path, scene_io.PROBE_DTYPE)
            elif base.startswith(("half_src", "sel", "sparse_valid", "sparse_anchor")):
                data[base] = np.fromfile(path, "<i4")
            else:
                data[base] = np.fromfile(path, "<f8")
    summary.update(case=name, src=spec["src"], args=[str(a) for a in args[3:]], size=list(spec["size"]),
                   generator="oracle/gen_golden.py via oracle/_ref/ref_parity gather (-ffp-contract=off)")
    with open(os.path.join(d, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    np.savez_compressed(os.path.join(d, "data.npz"), **data)
    print(name, {k: v.shape for k, v in data.items()})


def main():
    if not os.path.exists(REF):
        sys.exit("build oracle/_ref first: make -C oracle ref")
    names = sys.argv[1:] or list(CASES) + list(GATHER_CASES) + list(DYNAMIC_CASES) + list(RENDER_CASES)
    for n in names:
        if n in RENDER_CASES:
            build_render_case(n, RENDER_CASES[n])
        elif n in DYNAMIC_CASES:
            build_dynamic_case(n, DYNAMIC_CASES[n])
        elif n in GATHER_CASES:
            build_gather_case(n, GATHER_CASES[n])
        else:
            build_case(n, CASES[n])


if __name__ == "__main__":
    main()
