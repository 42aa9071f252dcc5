"""Debug helper: GPU ray records for chosen probes at a chosen pass of a golden case."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from golden_util import load  # noqa: E402
from paper_2007_14394_b200 import api  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

name, upto, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
probes = [int(x) for x in sys.argv[4:]]
case = load(name)
with Device(0, precision="f64") as dev:
    stage = api.ProbeStage(dev, case.scene, cfg=case.cfg(), res=case.res, spacing=case.spacing)
    for p in range(upto):
        stage.run_pass(p)
    stage.relocate_all()
    recs = dev.trace_debug(upto, stage.cfg, np.array([[0, i] for i in probes], np.int32))
    np.save(out, recs)
