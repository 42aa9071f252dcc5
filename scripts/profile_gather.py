"""Profiling driver: C2 volume after 3 passes, then a 1080p G-buffer, two gather
frames and composeFrame (the bench's C3 path), no timing. Used under ncu."""
import sys

sys.path.insert(0, ".")
from paper_2007_14394_b200 import api, scene_io  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
scene = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
with Device(0, precision=prec) as dev:
    stage = api.ProbeStage(dev, scene)
    for p in range(3):
        stage.run_pass(p)
    dev.render_gbuffer(scene.camera, 1920, 1080, stage.cfg)
    dev.gather(0, stage.cfg)
    dev.gather(1, stage.cfg)
    img, ms = dev.compose(stage.cfg)
    print("compose ms", ms)
