"""Helpers to load the committed golden fixtures (tests/golden/<case>/)."""
import json
import os

import numpy as np

from paper_2007_14394_b200 import scene_io

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(d for d in os.listdir(GOLDEN) if os.path.isdir(os.path.join(GOLDEN, d)))


class Case:
    def __init__(self, name):
        d = os.path.join(GOLDEN, name)
        self.name = name
        self.scene = scene_io.read_sdfs(os.path.join(d, "scene.sdfs"))
        with open(os.path.join(d, "summary.json")) as f:
            self.summary = json.load(f)
        with np.load(os.path.join(d, "data.npz")) as z:
            self.data = {k: z[k] for k in z.files}
        self.passes = self.summary["reps"][0]
        self.debug = self.summary["debug_probes"]
        args = self.summary["args"]
        self.res = None
        self.spacing = None
        self.n_rays = None
        self.budget = 0
        i = 0
        while i < len(args):
            a = args[i]
            if a == "--res":
                self.res = tuple(int(x) for x in args[i + 1:i + 4])
                i += 4
                continue
            if a == "--spacing":
                self.spacing = float(args[i + 1])
            elif a == "--nrays":
                self.n_rays = int(args[i + 1])
            elif a == "--budget":
                self.budget = int(args[i + 1])
            i += 2 if a in ("--spacing", "--nrays", "--passes", "--threads", "--debug-probe", "--budget") else 1
        self.levels = self.scene.cascade.levels

    def cfg(self):
        c = self.scene.cfg.copy()
        if self.n_rays is not None:
            c["n_rays_full"] = self.n_rays
        return c


def load(name):
    return Case(name)


GATHER_CASES = sorted(d for d in CASES if d.startswith("gather_"))
SCHED_CASES = sorted(d for d in CASES if d.startswith("sched_"))  # budgeted selectProbesForUpdate
DYNAMIC_CASES = sorted(d for d in CASES if d.startswith("dyn_"))  # C5 sequences
RENDER_CASES = sorted(d for d in CASES if d.startswith("render_"))  # Renderer::renderFrame loops
CASES = [d for d in CASES if not d.startswith(("gather_", "sched_", "dyn_", "render_"))]


class RenderCase:
    def __init__(self, name):
        d = os.path.join(GOLDEN, name)
        with open(os.path.join(d, "summary.json")) as f:
            self.summary = json.load(f)
        with np.load(os.path.join(d, "data.npz")) as z:
            self.data = {k: z[k] for k in z.files}
        self.frames = self.summary["frames"]
        self.w, self.h = self.summary["size"]
        self.scene_text = self.summary["scene_text"]
        args = self.summary["args"]
        self.n_rays = int(args[args.index("--nrays") + 1]) if "--nrays" in args else None


def load_render(name):
    return RenderCase(name)


class DynamicCase:
    """A C5 fixture: the authored scene text, every frame's active scene as the
    reference instantiated it, probes + atlas every `every` frames and on the last."""

    def __init__(self, name):
        d = os.path.join(GOLDEN, name)
        with open(os.path.join(d, "summary.json")) as f:
            self.summary = json.load(f)
        with np.load(os.path.join(d, "data.npz")) as z:
            self.data = {k: z[k] for k in z.files}
        self.frames = self.summary["frames"]
        self.scene_text = self.summary["scene_text"]
        args = self.summary["args"]
        self.n_rays = int(args[args.index("--nrays") + 1]) if "--nrays" in args else None
        self.dumped = sorted(int(k.split("_f")[1].split("_")[0]) for k in self.data if k.startswith("atlas_f")
                             and k.endswith("_c0"))


def load_dynamic(name):
    return DynamicCase(name)


class GatherCase:
    """A C3 fixture: probe passes of the source case, G-buffer, two gather frames."""

    def __init__(self, name):
        d = os.path.join(GOLDEN, name)
        with open(os.path.join(d, "summary.json")) as f:
            self.summary = json.load(f)
        with np.load(os.path.join(d, "data.npz")) as z:
            self.data = {k: z[k] for k in z.files}
        self.src = Case(self.summary["src"])
        self.scene = self.src.scene
        self.w, self.h = self.summary["size"]
        args = self.summary["args"]
        self.passes = int(args[args.index("--passes") + 1])
        self.frames = self.summary["frames"]


def load_gather(name):
    return GatherCase(name)
