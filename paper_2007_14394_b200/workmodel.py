"""Algorithmic-work model of the probe update for the roofline.

The tracing kernels are bound by the FP pipe, so ``roofline.achieved`` counts the
algorithmic FP instructions the reference's algorithm performs for the workload,
from the kernel's own event counters (TraceStats + evaluations by kind), weighted
by the per-event FP arithmetic instruction counts of SURVEY §8d (measured on
sm_100a SASS: FFMA/FADD/FMUL/FMNMX/FSETP/FSEL per event):

    AABB cluster test            14
    sphere / box / plane         7 / 15 / 6        (+9 when rotated: R^T q)
    cylinder / capsule           14 / 12            (+9 when rotated)
    min/select per evaluation    +2
    sphere-trace step            8   (p = o + d t, two compares, t += d)
    convolution (texel, ray)     7
    shadeHit per hit             400 (stencil: cascade/cell/trilinear weights, 8 probe
                                      loads, backface weights; 8 bilinear atlas lookups;
                                      direct light per light; the radiance sum)
    mvcWeightsHex call           2700 (12 triangles x ~215: 3 half-angle edges with
                                      their sqrt/asin polynomials, sin h and the three
                                      sin(h - theta_i) by angle addition, c_i/s_i, and
                                      three weight terms; + corner setup; the W_stencil
                                      term SURVEY §8d leaves to instrumentation)

The same counts are used for FP64 (DFMA/DADD/DMUL/DSETP; FP64 sqrt/div
sequences are counted as 1, i.e. the algorithmic count, not the issued one), so
``achieved`` is algorithmic instructions per second and ``peak`` the measured
FMA-instruction rate of that precision (sdfgi_measure_fp_peak).
"""
from __future__ import annotations

AABB = 14
EVAL = (7, 15, 6, 14, 12)  # sphere, box, plane, cylinder, capsule (unrotated)
ROTATE = 9
MINSEL = 2
STEP = 8
CONV = 7
SHADE = 400
MVC = 2700


def update_ops(stats, work, rays, texels_per_probe=64, shading=(0, 0)):
    """FP instructions of one update (or relocation: rays=0) from its counters;
    shading = (shadeHit calls, MVC evaluations) of the update."""
    tests = int(stats["clusters_visited"]) + int(stats["clusters_skipped"])
    evals = sum(int(w) for w in work[:5])
    ops = AABB * tests
    ops += sum(EVAL[k] * int(work[k]) for k in range(5))
    ops += ROTATE * int(work[5]) + MINSEL * evals
    ops += STEP * int(stats["trace_steps"])
    ops += CONV * texels_per_probe * int(rays)
    ops += SHADE * int(shading[0]) + MVC * int(shading[1])
    return ops
