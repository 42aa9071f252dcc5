"""Profiling driver: C2 scene, relocation, then one k_probe_update launch over every
`stride`-th probe (pass 0: 2N = 512 rays per probe). Used under ncu."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2007_14394_b200 import api, scene_io  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
stride = int(sys.argv[2]) if len(sys.argv) > 2 else 16
scene = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
with Device(0, precision=prec) as dev:
    stage = api.ProbeStage(dev, scene)
    stage.relocate_all()
    n = 32 * 16 * 32
    refs = np.array([[0, i] for i in range(0, n, stride)], np.int32)
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    for _ in range(reps):  # reps > 1: earlier calls warm up (lazy module loading), the last is reported
        res = dev.update(0, stage.cfg, refs)
        upd, _ = dev.last_kernel_ms()
    print(f"{prec} stride {stride}: {int(res['rays_traced'])} rays in {upd:.2f} ms "
          f"-> {int(res['rays_traced']) / upd / 1e6:.3f} Grays/s")
