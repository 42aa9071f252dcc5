"""C4 timing: 50k-primitive open scene, 128x32x128 probes, 256 rays, one bounce pass."""
import sys
import time

sys.path.insert(0, ".")
from paper_2007_14394_b200 import api, scenegen  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f32"
t0 = time.perf_counter()
scene = scenegen.with_fast_clusters(scenegen.c4_scene(50000), 8)
t1 = time.perf_counter()
with Device(0, precision=prec) as dev:
    stage = api.ProbeStage(dev, scene)
    t2 = time.perf_counter()
    print("accel", dev.accel_info(), f"scene gen+cluster {t1 - t0:.1f}s upload+grid {t2 - t1:.2f}s")
    for p in range(2):
        reps = stage.relocate_all()
        _, rel_ms = dev.last_kernel_ms()
        res = api.updateProbes(dev, stage.cfg, p)
        upd_ms, _ = dev.last_kernel_ms()
        dev.swap()
        print(prec, f"pass {p}: {int(res['rays_traced'])} rays in {upd_ms:.1f} ms "
              f"({int(res['rays_traced']) / upd_ms / 1e6:.3f} Grays/s), relocation {rel_ms:.1f} ms, dead {int(reps[0]['dead'])}")
