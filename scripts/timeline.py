"""Device timeline of bench steps (torch.profiler / CUPTI): kernel busy time vs
step span, and the largest idle gaps with the kernels either side.

    python scripts/timeline.py [f64|f32] [steps]

Writes gpurun_out/timeline_<prec>.json (summary) — timing under the profiler is
for locating gaps only, never a bench number."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2007_14394_b200.runtime import Device  # noqa: E402
from paper_2007_14394_b200 import api  # noqa: E402


def main():
    prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    dev = Device(0, precision=prec)
    scene = bench.load_workload("c2")[0]
    stage = api.ProbeStage(dev, scene)
    runner = bench.StepRunner(dev, stage)
    for _ in range(3):
        runner.fresh()
        runner.step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            runner.fresh()
            runner.step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev = sorted(ev, key=lambda e: e.time_range.start)
    spans = [(e.time_range.start, e.time_range.end, e.name) for e in ev]
    t0, t1 = spans[0][0], max(s[1] for s in spans)
    busy, last_end, gaps = 0.0, t0, []
    for s, e, n in spans:
        if s > last_end:
            gaps.append((s - last_end, prev, n))
        busy += max(0, e - max(s, last_end))
        last_end = max(last_end, e)
        prev = n
    gaps.sort(reverse=True)
    per = {}
    for st_, en, n in spans:
        per[n] = per.get(n, 0.0) + (en - st_)
    out = {"precision": prec, "steps": steps, "span_us": t1 - t0, "busy_us": busy,
           "idle_us": (t1 - t0) - busy, "n_device_ops": len(spans),
           "per_op_us": dict(sorted(((k[:90], v / steps) for k, v in per.items()), key=lambda kv: -kv[1])[:25]),
           "gaps_top": [{"us": g, "after": a[:80], "before": b[:80]} for g, a, b in gaps[:40]],
           "gap_hist": {k: sum(1 for g in gaps if lo <= g[0] < hi)
                        for k, lo, hi in (("<5us", 0, 5), ("5-20us", 5, 20), ("20-100us", 20, 100),
                                          (">=100us", 100, 1e12))}}
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/timeline_{prec}.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("gaps_top", "per_op_us")}))
    for k, v in out["per_op_us"].items():
        print(f"{v:9.1f} us/step  {k}")
    for g in out["gaps_top"][:20]:
        print(f"{g['us']:8.1f} us  after {g['after']}  before {g['before']}")


if __name__ == "__main__":
    main()
