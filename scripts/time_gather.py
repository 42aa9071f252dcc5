"""Warm device timing of one 1080p gather frame + compose on the C2 volume."""
import sys

sys.path.insert(0, ".")
from paper_2007_14394_b200 import api, scene_io  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
scene = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
accel = int(sys.argv[2]) if len(sys.argv) > 2 else 2
with Device(0, precision=prec) as dev:
    dev.set_accel(accel)
    stage = api.ProbeStage(dev, scene)
    for p in range(3):
        stage.run_pass(p)
    dev.render_gbuffer(scene.camera, 1920, 1080, stage.cfg)
    for f in range(4):
        dev.gather(f, stage.cfg)
        _, cms = dev.compose(stage.cfg, download=False)
    st = dev.last_gather_ms()
    print(f"{prec} accel {accel} gather {sum(st):.2f} ms (contact {st[3]:.2f}) compose {cms:.2f} ms")
