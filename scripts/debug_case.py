"""Debug helper: replay a golden case on the GPU and report per-pass texel errors."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from golden_util import load  # noqa: E402
from paper_2007_14394_b200 import api  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

name = sys.argv[1]
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
case = load(name)
out = {}
with Device(0, precision=prec) as dev:
    stage = api.ProbeStage(dev, case.scene, cfg=case.cfg(), res=case.res, spacing=case.spacing)
    for p in range(len(case.passes)):
        stage.run_pass(p)
        for level in range(stage.levels):
            got = dev.atlas(level, 0).astype(np.float64)
            wa = case.data[f"atlas_p{p}_c{level}"].astype(np.float64)
            floor = 0.05 * max(float(np.mean(np.abs(wa))), 1e-12)
            err = np.abs(got - wa) / np.maximum(np.abs(wa), floor)
            per_probe = err.reshape(len(err), -1).max(axis=1)
            worst = np.argsort(per_probe)[::-1][:10]
            out[f"p{p}_c{level}"] = {
                "max": float(err.max()), "n_bad": int((err > 1e-3).sum()), "n_exact": int((got == wa).sum()),
                "n": int(err.size), "worst_probes": worst.tolist(), "worst_err": per_probe[worst].tolist(),
                "bad_probes": int((per_probe > 1e-3).sum()),
            }
print(json.dumps(out, indent=1))
