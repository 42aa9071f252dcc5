"""Measure the per-event FP instruction weights of the shading kernels (SURVEY §8d:
"MVC call ~2-3k, count once instrumented") and the executed FP instructions of
every update kernel, for the roofline's algorithmic-work model (workmodel.py).

  python scripts/measure_fp_ops.py run <prec> <out.json>
      one C2 step with counters (event counts per pass: shadeHit calls, MVC calls,
      K1/K2 query events) -> out.json
  ncu --metrics <FP op metrics> --csv --log-file <csv> python scripts/measure_fp_ops.py run <prec> /dev/null
      the same step under ncu -> executed FP thread instructions per kernel launch
  python scripts/measure_fp_ops.py summarize <prec> <counts.json> <ncu.csv> <weights.json>
      weights = executed FP instructions of K3a (K3c) / shadeHit (MVC) calls; plus the
      executed counts of every kernel, for comparison with the SASS-weighted model
"""
import csv
import json
import re
import sys

sys.path.insert(0, ".")

OPS = {"f64": ("dadd", "dmul", "dfma"), "f32": ("fadd", "fmul", "ffma")}
METRICS = ",".join(["gpu__time_duration.sum"] + [f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum"
                                                  for ops in OPS.values() for o in ops])


def run(prec, out):
    from paper_2007_14394_b200 import api, scene_io
    from paper_2007_14394_b200.runtime import Device

    scene = scene_io.read_sdfs("paper_2007_14394_b200/data/c2.sdfs")
    passes = []
    with Device(0, precision=prec) as dev:
        stage = api.ProbeStage(dev, scene)
        for p in range(3):
            stage.relocate_all()
            res, st = api.updateProbes(dev, stage.cfg, p, None, stats=True)
            passes.append({"rays": int(res["rays_traced"]), "shading": dev.last_shading_work(),
                           "trace": dev.last_trace_counters()})
            dev.swap()
    if out != "/dev/null":
        json.dump({"precision": prec, "passes": passes}, open(out, "w"), indent=1)


def summarize(prec, counts, ncu_csv, out):
    c = json.load(open(counts))
    rows = [r for r in csv.reader(open(ncu_csv)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = {}
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("sdfgi_dev::", "")
        d = launches.setdefault(int(r[ii]), {"kernel": name})
        try:
            d[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    # FP64 mode: the FP64 pipe's instructions; FP32 mode: both (its shading sums stay FP64)
    ops = OPS["f64"] if prec == "f64" else OPS["f32"] + OPS["f64"]
    fp = lambda d: sum(d.get(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum", 0.0) for o in ops)  # noqa
    per = {}
    for lid in sorted(launches):
        d = launches[lid]
        k = per.setdefault(d["kernel"], {"launches": 0, "fp_thread_inst": 0.0, "ns": 0.0})
        k["launches"] += 1
        k["fp_thread_inst"] += fp(d)
        k["ns"] += d.get("gpu__time_duration.sum", 0.0)
    shade_calls = sum(p["shading"][0] for p in c["passes"])
    mvc_calls = sum(p["shading"][1] for p in c["passes"])
    k3a = next(v for k, v in per.items() if k.startswith("k_shade_rays"))
    k3c = next(v for k, v in per.items() if k.startswith("k_shade_mvc"))
    res = {
        "precision": prec,
        "source": {"counts": counts, "ncu_launch_list": ncu_csv,
                   "metrics": [f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum" for o in ops]},
        "shade_calls_per_step": shade_calls,
        "mvc_calls_per_step": mvc_calls,
        # executed FP instructions per event: what the shading kernels issue per call
        "SHADE": k3a["fp_thread_inst"] / max(shade_calls, 1),
        "MVC": k3c["fp_thread_inst"] / max(mvc_calls, 1),
        "executed_fp_thread_inst_per_kernel": per,
    }
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: res[k] for k in ("SHADE", "MVC", "shade_calls_per_step", "mvc_calls_per_step")}))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3])
    else:
        summarize(*sys.argv[2:6])
