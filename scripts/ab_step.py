"""A/B timing of the C2 step (3 passes, device events, L2 flushed) for library
variants: python scripts/ab_step.py [prec] [reps] ; SDFGI_LIB selects the build."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2007_14394_b200 import api, runtime, scene_io  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402

if os.environ.get("SDFGI_LIB"):  # an older variant may lack newer entry points
    import ctypes

    _probe = ctypes.CDLL(os.environ["SDFGI_LIB"])
    runtime._SIGS = {k: v for k, v in runtime._SIGS.items() if hasattr(_probe, k)}
fused = os.environ.get("FUSED") == "1"  # one sdfgi_probe_stage call per pass
queued = os.environ.get("ASYNC") == "1"  # sdfgi_probe_stage_async per pass, one collect per step

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
scene = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
with Device(0, precision=prec) as dev:
    stage = api.ProbeStage(dev, scene)
    ext = torch.cuda.ExternalStream(dev.stream)
    per_pass, steps = [], []
    for r in range(reps + 2):
        for lv in range(stage.levels):
            dev.reset_probes(lv)
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        pp = []
        for p in range(3):
            if queued:
                dev.probe_stage_async(p, stage.cfg)
            elif fused:
                dev.probe_stage(p, stage.cfg)
            else:
                stage.relocate_all()
                api.updateProbes(dev, stage.cfg, p)
            pp.append(0.0 if queued else dev.last_kernel_ms()[0])
            dev.swap()
        if queued:
            dev.probe_stage_collect()
        e1.record(ext)
        e1.synchronize()
        if r >= 2:
            steps.append(e0.elapsed_time(e1))
            per_pass.append(pp)
    pp = np.median(np.array(per_pass), axis=0)
    lib = os.environ.get("SDFGI_LIB", "cur").split("/")[-2] if os.environ.get("SDFGI_LIB") else "cur"
    lib += "+async" if queued else ("+fused" if fused else "")
    print(f"{lib:12s} {prec} step {np.median(steps):7.2f} ms  passes " + " ".join(f"{x:6.2f}" for x in pp))
