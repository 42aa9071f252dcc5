"""Algorithmic-work model of the probe update for the roofline.

The tracing and shading kernels are bound by the FP pipe, so ``roofline.achieved``
counts the FP instructions of the reference's algorithm for the workload, from the
kernels' own event counters (TraceStats + evaluations by kind, per tracing kernel),
each event weighted by a measured FP instruction count:

* per query event, SURVEY §8d's SASS weights (FFMA/FADD/FMUL/FMNMX/FSETP/FSEL
  counted per event on sm_100a; Appendix A of SURVEY.md):

      AABB cluster test            14
      sphere / box / plane         7 / 15 / 6        (+9 when rotated: R^T q)
      cylinder / capsule           14 / 12            (+9 when rotated)
      min/select per evaluation    +2
      sphere-trace step            8   (p = o + d t, two compares, t += d)
      convolution (texel, ray)     7

* per shading event, "count once instrumented": the FP instructions
  the shading kernels execute per call, measured with ncu
  (smsp__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum, FP32 mode
  also {fadd,fmul,ffma}) over a C2 step, divided by the calls counted by the
  kernels: SHADE per shadeHit call (K3a: direct light in light order, the
  trilinear stencil, backface weights, 8 bilinear lookups) and MVC per mean-value
  lookup (K3c: mvcWeightsHex + the lookup). The measurement is committed as
  profiles/r0*_fp_weights_<prec>_v*.json (scripts/gpu_fp_weights.sh); the newest
  is used.

``achieved`` is algorithmic instructions per second and ``peak`` the measured
FMA-instruction rate of that precision (sdfgi_measure_fp_peak).
"""
from __future__ import annotations

import glob
import json
import os
import re

AABB = 14
EVAL = (7, 15, 6, 14, 12)  # sphere, box, plane, cylinder, capsule (unrotated)
ROTATE = 9
MINSEL = 2
STEP = 8
CONV = 7

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def shading_weights(precision="f64"):
    """(SHADE, MVC, source file) from the newest committed measurement."""
    best = None
    for f in glob.glob(os.path.join(_ROOT, "profiles", f"r*_fp_weights_{precision}_v*.json")):
        m = re.search(r"r(\d+)_fp_weights_\w+_v(\d+)\.json$", f)
        if m and (best is None or (int(m.group(1)), int(m.group(2))) > best[0]):
            best = ((int(m.group(1)), int(m.group(2))), f)
    if best is None:
        raise RuntimeError(f"no profiles/r*_fp_weights_{precision}_v*.json: run scripts/gpu_fp_weights.sh")
    d = json.load(open(best[1]))
    return float(d["SHADE"]), float(d["MVC"]), os.path.relpath(best[1], _ROOT)


def query_ops(stats, work):
    """FP instructions of the SDF queries and march steps behind a set of counters."""
    tests = int(stats["clusters_visited"]) + int(stats["clusters_skipped"])
    evals = sum(int(w) for w in work[:5])
    ops = AABB * tests
    ops += sum(EVAL[k] * int(work[k]) for k in range(5))
    ops += ROTATE * int(work[5]) + MINSEL * evals
    ops += STEP * int(stats["trace_steps"])
    return ops


def convolve_ops(rays, texels_per_probe=64):
    return CONV * texels_per_probe * int(rays)


def shading_ops(shading, precision="f64"):
    shade, mvc, _ = shading_weights(precision)
    return shade * int(shading[0]) + mvc * int(shading[1])


def update_ops(stats, work, rays, texels_per_probe=64, shading=(0, 0), precision="f64"):
    """FP instructions of one update (or relocation: rays=0) from its counters;
    shading = (shadeHit calls, MVC evaluations) of the update."""
    ops = query_ops(stats, work) + convolve_ops(rays, texels_per_probe)
    if shading[0] or shading[1]:
        ops += shading_ops(shading, precision)
    return ops
