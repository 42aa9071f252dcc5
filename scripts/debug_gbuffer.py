"""FP32 vs FP64 device G-buffer on C2 (depth/prim agreement + timing)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2007_14394_b200 import api, scene_io  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

scene = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
out = {}
for prec in ("f64", "f32"):
    with Device(0, precision=prec) as dev:
        stage = api.ProbeStage(dev, scene)
        for rep in range(2):
            t0 = time.perf_counter()
            dev.render_gbuffer(scene.camera, 1920, 1080, stage.cfg)
            dt = time.perf_counter() - t0
        out[prec] = dev.gbuffer()
        print(prec, f"{dt * 1e3:.1f} ms", "sky", int(np.sum(~np.isfinite(out[prec]["depth"]))))
a, b = out["f64"], out["f32"]
geo = np.isfinite(a["depth"]) & np.isfinite(b["depth"])
print("sky mismatch", int(np.sum(np.isfinite(a["depth"]) != np.isfinite(b["depth"]))))
print("prim match", float(np.mean(a["prim_index"][geo] == b["prim_index"][geo])))
print("depth rel err max", float(np.max(np.abs(a["depth"][geo] - b["depth"][geo]) / a["depth"][geo])))
