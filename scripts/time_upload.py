"""Scene upload (acceleration build) time: C2 and C4, each uploaded twice with
different geometry (the second build is timed warm)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2007_14394_b200 import scene_io, scenegen  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

c2 = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
c4 = scenegen.with_fast_clusters(scenegen.c4_scene(50000), 8)
with Device(0, precision="f64") as dev:
    for name, sc in (("C2", c2), ("C4", c4)):
        for rep in range(2):
            sc.prims["trans"][1, 0] += 1e-6  # new geometry: no cached acceleration
            t0 = time.perf_counter()
            dev.upload_scene(sc)
            dt = time.perf_counter() - t0
        print(f"{name}: upload + grid/BVH build {dt * 1e3:.1f} ms, {dev.accel_info()}")
