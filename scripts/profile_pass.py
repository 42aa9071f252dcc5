"""Profiling driver: the C2 step's first `passes` passes (default 2), so the later
passes' kernels (bounce lookups, K3c) can be captured with ncu --launch-skip."""
import sys

sys.path.insert(0, ".")
from paper_2007_14394_b200 import api, scene_io  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
scene = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
with Device(0, precision=prec) as dev:
    stage = api.ProbeStage(dev, scene)
    for p in range(passes):
        stage.run_pass(p)
    print("ok", dev.launch_count())
