"""Wall-clock phases of bench.py's e2e step (C2, FP64): scene upload, probe
reset + upload (pinned), the 3 passes, the atlas download (pinned). Each phase
ends with a device synchronisation. python scripts/e2e_phases.py [steps]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2007_14394_b200 import api, scene_io  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
scene = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
with Device(0, precision="f64") as dev:
    stage = api.ProbeStage(dev, scene)
    n = int(np.prod(scene.cascade.res))
    t = dev.oct_res + 2
    pin = torch.empty(n * scene_io.PROBE_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
    probes_host = pin.numpy().view(scene_io.PROBE_DTYPE)
    stage.reset()
    probes_host[:] = dev.probes(0)
    atlas_pin = torch.empty(n * t * t * 3, dtype=torch.float32, pin_memory=True)
    atlas_host = atlas_pin.numpy().reshape(n, t, t, 3)
    ph = {k: [] for k in ("upload_scene", "reset+upload_probes", "passes", "download", "total")}
    for i in range(steps + 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.upload_scene(scene)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        dev.reset_probes(0)
        dev.upload_probes(0, probes_host)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for p in range(3):
            stage.run_pass(p)
        t3 = time.perf_counter()
        dev.atlas(0, 0, out=atlas_host)
        t4 = time.perf_counter()
        if i >= 2:
            for k, v in zip(ph, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
                ph[k].append(v * 1e3)
    for k, v in ph.items():
        print(f"{k:22s} {np.median(v):8.3f} ms")
