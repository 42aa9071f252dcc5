#!/usr/bin/env python3
"""Benchmark: SDFDDGI per-frame probe update on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): the ~2k-primitive synthetic
Sponza-scale scene (paper_2007_14394_b200/data/c2.sdfs, clusters built by the
reference's buildClusters), a 32x16x32 probe volume at spacing 0.45, 256 rays per
probe, 3 bounces. One step = a fresh probe volume taken through 3 passes
(frames 0, 1, 2), each pass = relocation (d) + the batched probe update (a,b,c)
reading the previous pass's atlas + the atlas swap. Pass 0 traces 2N rays per
probe (fresh probes reject history, probe_update.hpp:173).

  value        Grays/s = probe rays (sum of raysTraced) / device time of the step,
               inputs resident in HBM, CUDA events on the context's stream, L2
               flushed (256 MB write) before every timed step, max over ranks.
  e2e          same metric through the public API with host buffers: scene upload,
               fresh-probe upload from pinned host memory, 3 passes, atlas download
               into pinned host memory, all inside the timed region (wall clock).
  roofline     dominant kernel k_probe_update: algorithmic FP instructions
               (workmodel.py x the kernel's own counters) / its event-timed
               duration, against the FMA-pipe rate measured live on this GPU.
  cpu_baseline the reference itself (oracle/_ref, compiled from /root/reference)
               on the host's cores over a bounded sample of the same workload.

--impl reference runs only the CPU reference arm (rank 0), on the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2007_14394_b200 import scene_io, workmodel  # noqa: E402

C2_PATH = os.path.join(ROOT, "paper_2007_14394_b200", "data", "c2.sdfs")
PASSES = 3
METRIC = "probe-update Grays/s & ms/frame (32x16x32 probes, 256 rays)"
UNIT = "Grays/s"


def latest_profiles(stem, ext):
    """profiles/r<round>_<stem>_v<version>.<ext>, oldest first: sorted by (round,
    version) numerically, so v12 sorts after v9 and r02 after r01."""
    import glob

    out = []
    for f in glob.glob(os.path.join(ROOT, "profiles", f"r*_{stem}_v*.{ext}")):
        m = re.search(rf"r(\d+)_{re.escape(stem)}_v(\d+)\.{ext}$", os.path.basename(f))
        if m:
            out.append(((int(m.group(1)), int(m.group(2))), f))
    return [f for _, f in sorted(out)]


STEP_KERNELS = ("k_relocate", "k_ray_setup", "k_ray_scan", "k_trace_primary", "k_trace_shadow", "k_shade_rays",
                "k_convolve")


def ncu_kernel_traffic(precision, kernel_group):
    """DRAM bytes (read + write) per launch of the dominant kernel group from the
    newest committed `ncu --set full` summary (profiles/r*_ncu_step_<prec>_v*.json):
    the capture replays one C2 pass, so per launch = per pass."""
    files = latest_profiles(f"ncu_step_{precision}", "json")
    if not files:
        return None, None
    caps = json.load(open(files[-1])).get("full_captures", [])
    names = kernel_group.split("+")
    tot, seen = 0.0, False
    for c in caps:
        name = re.sub(r"\(.*", "", c.get("Kernel Name", "")).replace("void ", "")
        if any(n in name for n in names):
            try:
                tot += float(c["dram__bytes_read.sum"]) + float(c["dram__bytes_write.sum"])
                seen = True
            except (KeyError, ValueError):
                continue
    return (tot if seen else None), os.path.relpath(files[-1], ROOT)


def ncu_step_traffic(precision):
    """DRAM bytes (read + write) of one C2 step's update kernels from the committed ncu
    launch list of scripts/profile_step.py (profiles/r01_step_launches_<prec>_v*.csv,
    the newest): kernels launched before the gather's first k_render_gbuffer."""
    import csv
    import glob

    files = latest_profiles(f"step_launches_{precision}", "csv")
    if not files:
        return None, None
    rows = [r for r in csv.reader(open(files[-1])) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    total, seen_gather = 0.0, False
    for r in sorted(rows[1:], key=lambda r: int(r[ii])):
        name = r[ki]
        if "k_render_gbuffer" in name:
            seen_gather = True
        if seen_gather or not any(k in name for k in STEP_KERNELS):
            continue
        if r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total += float(r[vi].replace(",", ""))
    return total, os.path.relpath(files[-1], ROOT)


# Memory-side kernels reported against the HBM roofline. k_convolve (the atlas
# blend) is not among them: its 64-texel x n-ray cosine sums keep the FP64 pipe
# ~77% busy (profiles/r01_ncu_step_f64_v6.json) while it moves 2 KB per probe.
HBM_KERNELS = ("k_downsample", "k_select", "k_resolve", "k_contact_combine", "k_compose")


def ncu_pipe_kernels(precision):
    """Per-kernel pipe utilisation of the hot update kernels from the committed
    `ncu --set full` capture summary (profiles/r01_ncu_step_<prec>_v*.json, newest):
    the FP64 / FMA pipe cycles active, issue slots busy and active threads per
    issued instruction (the divergence that bounds the tracing kernels)."""
    import glob

    files = latest_profiles(f"ncu_step_{precision}", "json")
    if not files:
        return None
    caps = json.load(open(files[-1])).get("full_captures", [])
    out = {}
    for c in caps:
        name = re.sub(r"\(.*", "", c.get("Kernel Name", "")).replace("void ", "")
        try:
            out[name] = {
                "ms": float(c["gpu__time_duration.sum"]),
                "fp64_pipe_pct": float(c["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
                "fma_pipe_pct": float(c["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]),
                "issue_active_pct": float(c["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
                "threads_per_inst": float(c["smsp__thread_inst_executed_per_inst_executed.ratio"]),
            }
        except (KeyError, ValueError):
            continue
    return {"source": os.path.relpath(files[-1], ROOT), "kernels": out}


def ncu_hbm_kernels(precision, hbm_peak):
    """Achieved DRAM GB/s of the memory-side kernels (atlas blend, gather stages)
    from the committed ncu launch list: (read + write bytes) / duration per launch,
    averaged over launches (cold-cache, serialised: a lower bound on the bench's)."""
    import csv
    import glob

    files = latest_profiles(f"step_launches_{precision}", "csv")
    if not files:
        return None
    rows = [r for r in csv.reader(open(files[-1])) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        name = next((k for k in HBM_KERNELS if k in r[ki]), None)
        if name is None:
            continue
        d = per.setdefault(name, {}).setdefault(r[ii], {})
        d[r[mi]] = float(r[vi].replace(",", ""))
    out = {}
    for name, launches in per.items():
        gbs = [(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / v["gpu__time_duration.sum"]
               for v in launches.values() if v.get("gpu__time_duration.sum")]
        if gbs:
            a = sum(gbs) / len(gbs)
            out[name] = {"achieved_gbs": a, "peak_gbs": hbm_peak, "frac": a / hbm_peak, "launches": len(gbs)}
    return {"source": os.path.relpath(files[-1], ROOT), "kernels": out}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# ------------------------------------------------------------------ CPU reference
def ref_binary():
    """The reference compiled from /root/reference by oracle/Makefile (travels in-tree)."""
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        flags = ""
    names = (["ref_perf_v4"] if "avx512f" in flags else []) + ["ref_perf_v3"]
    for n in names:
        p = os.path.join(ROOT, "oracle", "_ref", n)
        if os.path.exists(p):
            return p
    return None


def workload_sdfs(config):
    """The workload's scene as an SDFS file the reference driver reads (C4 is
    generated, then written to a temporary file)."""
    if config == "c2":
        return C2_PATH
    import tempfile

    scene, _ = load_workload(config)
    path = os.path.join(tempfile.gettempdir(), f"sdfgi_bench_{config}.sdfs")
    scene_io.write_sdfs(path, scene)
    return path


CPU_STRIDE = {"c2": 7, "c4": 2039}  # coprime with the grid dims: every x, y, z column is sampled


def cpu_reference_sample(stride, threads, reps=1, sdfs=C2_PATH):
    """Run the reference probe stage (pipeline.hpp:108-151) for PASSES passes on every
    `stride`-th probe. Returns per-rep (rays, seconds) with relocation time scaled to the
    sampled fraction (relocation always runs on the whole volume)."""
    exe = ref_binary()
    if exe is None:
        return None, "oracle/_ref not built"
    cmd = [exe, "passes", sdfs, os.devnull, "--passes", str(PASSES), "--threads", str(threads),
           "--stride", str(stride), "--reps", str(reps), "--no-dump"]
    r = subprocess.run(cmd, capture_output=True, text=True, check=True)
    out = json.loads(r.stdout)
    res = []
    for rep in out["reps"]:
        rays = sum(p["rays_traced"] for p in rep)
        secs = sum(p["update_ms"] + p["reloc_ms"] / stride for p in rep) / 1e3
        res.append((rays, secs))
    return res, os.path.basename(exe)


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ our arm
def load_workload(config):
    """C2 (BASELINE configs[1], the headline) or C4 (configs[3]: ~50k primitives,
    128x32x128 probes at spacing 1.875, clusters from the library's linear-time
    builder)."""
    if config == "c2":
        return scene_io.read_sdfs(C2_PATH), WORKLOADS["c2"]
    from paper_2007_14394_b200 import scenegen

    return scenegen.with_fast_clusters(scenegen.c4_scene(50000), 8), WORKLOADS["c4"]


WORKLOADS = {
    "c2": "C2: ~2k-primitive synthetic Sponza-scale SDF scene, 32x16x32 probes, 256 rays, 3 bounces, relocation each pass",
    "c4": "C4: ~50k-primitive open synthetic scene, 128x32x128 probes, 256 rays, 3 bounces, relocation each pass",
}


class StepRunner:
    """One step = a fresh probe volume (makeCascade state) taken through PASSES
    passes (frames 0..PASSES-1): relocation + batched update + swap per pass."""

    def __init__(self, dev, stage):
        self.dev, self.stage = dev, stage

    def fresh(self):
        for level in range(self.stage.levels):
            self.dev.reset_probes(level)
        self.dev.stage_ms_sum(reset=True)

    def step(self, stats=False):
        """-> rays, update-kernel ms, per-stage ms (summed over passes), and with
        stats the algorithmic work per kernel (workmodel) and the raw counters."""
        from paper_2007_14394_b200 import api

        dev, stage = self.dev, self.stage
        rays, work_all = 0, []
        work = dict.fromkeys(("k1", "k2", "shade", "convolve"), 0.0)
        prec = dev.precision
        for p in range(PASSES):
            if not stats:  # the probe stage of pipeline.hpp:108-151 queued (one sync per step, below)
                dev.probe_stage_async(p, stage.cfg)
                dev.swap()
                continue
            # relocation and update counters apart: one call each
            stage.relocate_all(stats=True)
            res, st = api.updateProbes(dev, stage.cfg, p, None, stats=True)
            tc = dev.last_trace_counters()
            sh = dev.last_shading_work()
            work["k1"] += workmodel.query_ops(*tc["k1"])
            work["k2"] += workmodel.query_ops(*tc["k2"])
            work["shade"] += workmodel.shading_ops(sh, prec)
            work["convolve"] += workmodel.convolve_ops(int(res["rays_traced"]))
            work_all.append({"k1": tc["k1"], "k2": tc["k2"], "shading": sh})
            rays += int(res["rays_traced"])
            dev.swap()
        if not stats:  # the step's passes, their results read back
            _, results = dev.probe_stage_collect()
            rays = int(results["rays_traced"].sum())
        # every pass's stage events, summed on the device side (read once per step)
        stage_ms, upd_ms = dev.stage_ms_sum(reset=True)
        return rays, upd_ms, stage_ms, work, work_all


KERNEL_STAGES = {
    # stage group -> (kernels, stages of last_stage_ms, work key)
    "k_trace_primary": ("K1 primary rays, near + far phase (sphereTrace)", ("k1", "k1_far"), "k1"),
    "k_trace_shadow": ("K2 shadow rays, near + far phase (softShadowTrace)", ("k2", "k2_far"), "k2"),
    "k_shade_rays+k_shade_mvc": ("K3a + K3c (shadeHit, bounce lookup with MVC)", ("shade",), "shade"),
    "k_convolve": ("K3b (convolveIrradiance + hysteresis blend + border)", ("convolve",), "convolve"),
}


def roofline_of(args, dev, kern, ms_step, work_step, n_probes):
    """Per-kernel rooflines of the update: algorithmic FP instructions (workmodel.py,
    from the kernels' own counters; shading weights measured with ncu) / the
    kernel's device time (CUDA events around each stage on the context's stream,
    median over the timed steps), against the measured FMA-instruction rate. The
    headline object is the dominant kernel (largest share of the step)."""
    f64_rate, f32_rate = dev.measure_fp_peak()
    peak_rate = f64_rate if args.precision == "f64" else f32_rate
    upd_ms = statistics.median(k[0] for k in kern)
    stage_ms = {k: statistics.median(s[1][k] for s in kern) for k in kern[0][1]}
    kernels = {}
    for name, (what, stages, wk) in KERNEL_STAGES.items():
        ms = sum(stage_ms[st] for st in stages)
        ach = work_step[wk] / (ms * 1e-3) if ms > 0 else 0.0
        kernels[name] = {"what": what, "ms_per_step": ms, "share_of_step": ms / ms_step,
                         "work_instr_per_step": work_step[wk], "achieved": ach / 1e12, "frac": ach / peak_rate}
    total_work = sum(work_step.values())
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    traffic, traffic_src = ncu_kernel_traffic(args.precision, dom) if args.config == "c2" else (None, None)
    _, _, wsrc = workmodel.shading_weights(args.precision)
    return {
        "bound": "fp64" if args.precision == "f64" else "fp32",
        "kernel": dom,
        "achieved": kernels[dom]["achieved"],
        "peak": peak_rate / 1e12,
        "unit": "Tinstr/s",
        "frac": kernels[dom]["frac"],
        "traffic": traffic,
        "traffic_unit": "DRAM bytes per launch of the dominant kernel (ncu --set full capture, cold cache)",
        "traffic_source": traffic_src,
        "algorithmic_instr_per_launch": kernels[dom]["work_instr_per_step"] / PASSES,
        "kernels": kernels,
        "wavefront_total": {"ms_per_step": upd_ms, "work_instr_per_step": total_work,
                            "achieved": total_work / (upd_ms * 1e-3) / 1e12,
                            "frac": total_work / (upd_ms * 1e-3) / peak_rate, "share_of_step": upd_ms / ms_step},
        "algorithmic_hbm_bytes_per_step": PASSES * n_probes * (768 + 1200),
        "peak_source": "measured live: sdfgi_measure_fp_peak FMA-instruction rate (MEASURED_PEAKS.json has no FP "
                       "pipe entry)",
        "work_model": f"paper_2007_14394_b200/workmodel.py; query weights SURVEY §8d SASS counts, shading weights "
                      f"{wsrc}",
    }


def timed_steps(runner, steps, ext, flush, torch, barrier):
    """Device time of `steps` fresh steps (CUDA events on the context's stream, L2
    flushed before each): per-step ms, update-kernel ms and rays."""
    times, kern, rays = [], [], 0
    barrier()
    torch.cuda.synchronize()
    for _ in range(steps):
        runner.fresh()
        flush.fill_(1.0)  # L2 flush (256 MB > 126 MB L2) outside the timed window
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        rays, upd_ms, stage_ms, _, _ = runner.step()
        e1.record(ext)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        kern.append((upd_ms, stage_ms))
    barrier()
    torch.cuda.synchronize()
    return times, kern, rays


def max_over_ranks(x, dist, torch):
    if dist is None:
        return x
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2007_14394_b200 import api
    from paper_2007_14394_b200.runtime import Device, nccl_unique_id

    torch.cuda.set_device(local_rank)
    uid = None
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the init lines let a reader count the ranks
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    scene, workload = load_workload(args.config)
    n_probes = int(np.prod(scene.cascade.res))
    dev = Device(local_rank, rank, world, uid, precision=args.precision)
    stage = api.ProbeStage(dev, scene)
    runner = StepRunner(dev, stage)
    ext = torch.cuda.ExternalStream(dev.stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()

    # algorithmic work of one step (untimed stats run: counters cost registers/atomics)
    runner.fresh()
    rays_stats, _, _, work_step, work_all = runner.step(stats=True)
    for _ in range(args.warmup):
        runner.fresh()
        runner.step()
    torch.cuda.synchronize()
    launches0 = dev.launch_count()
    with ClockSampler(local_rank) as clk:
        times, kern, rays_step = timed_steps(runner, args.steps, ext, flush, torch, barrier)
    launches = dev.launch_count() - launches0
    total_ms = max_over_ranks(sum(times), dist, torch)
    ms_step = total_ms / args.steps
    value = rays_step * args.steps / (total_ms * 1e-3) / 1e9

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e_val, h2d, d2h = e2e_run(args, dev, stage, scene, barrier, dist, torch)
    gather = None
    if not args.no_gather and args.config == "c2":
        gather = gather_bench(args, dev, stage, scene, torch, ext, flush)

    roofline = roofline_of(args, dev, kern, ms_step, work_step, n_probes)
    hbm_peak = float(load_peaks().get("hbm_gbs", 7700.0))
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": args.precision,
        "data": f"synthetic (deterministic {args.config.upper()} scene, SURVEY §8d; no network)",
        "config": {
            "workload": workload,
            "primitives": int(len(scene.prims)),
            "clusters": int(len(scene.clusters)),
            "probes": n_probes,
            "probe_grid": list(map(int, scene.cascade.res)),
            "rays_per_probe": int(stage.cfg["n_rays_full"][0]),
            "bounces": PASSES,
            "rays_per_step": rays_step,
            "parallelism": f"z-slab x{world}" if world > 1 else "single GPU",
            "l2": "flushed (256 MB write) before every timed step",
            "precision_mode": args.precision,
            "cluster_walk": dev.accel_info(),
        },
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "scene re-uploaded every step; the candidate grid is rebuilt only when the geometry "
                        "changes (static scene: kept)"},
        "gpu_launches": launches,
        "roofline": roofline,
        "clocks": clk.summary(),
        "algorithmic_counters_step": work_all,
    }
    if args.config == "c2":
        line["roofline_hbm_kernels"] = ncu_hbm_kernels(args.precision, hbm_peak)
        line["pipe_kernels_ncu"] = ncu_pipe_kernels(args.precision)
        line["gather_c3"] = gather
        line["frame_ms_update_plus_gather"] = (ms_step + gather["ms_per_frame"]) if gather else None
        line["frame_ms_update_gather_compose"] = (ms_step + gather["ms_per_frame"] + gather["compose_ms"]) \
            if gather else None
    if world > 1:
        line["atlas_equal_1gpu"] = atlas_equal_1gpu(dev, stage, runner, scene, rank, local_rank, dist, torch)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == "c2":
        line["cpu_baseline"] = cpu_baseline(rays_step)
    if not args.no_alt:
        # the other arithmetic mode on the same workload, same timing rules (the
        # headline stays FP64 = the reference's own precision, bit-exact decisions)
        alt = "f32" if args.precision == "f64" else "f64"
        dev.set_precision(alt)
        runner.fresh()
        runner.step()
        times_alt, _, r_alt = timed_steps(runner, args.steps, ext, flush, torch, barrier)
        ms_alt = max_over_ranks(sum(times_alt) / len(times_alt), dist, torch)
        line["alt_precision"] = {
            "dtype": alt, "value": r_alt / (ms_alt * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms_alt,
            "texel_error_vs_oracle": "FP32: error distribution over the whole C2 step printed by "
                                     "tests/test_gpu_oracle.py::test_c2_f32_mode_error_report" if alt == "f32" else
                                     "FP64: bit-exact relocation and directions; every texel within 1e-3 "
                                     "(tests/test_gpu_oracle.py::test_c2_full_step_matches_oracle)",
        }
        dev.set_precision(args.precision)
    if not args.no_c4 and args.config == "c2":
        line["c4"] = c4_bench(args, rank, world, local_rank, uid, ext, flush, torch, barrier, dist)
        if world == 1:
            line["c5_animated"] = c5_bench(args, local_rank, torch)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dev.close()
    if dist is not None:
        dist.destroy_process_group()


def animated(scene, frame, ids):
    """C2 with primitives `ids` on small orbits at `frame` (cluster boxes grown to
    keep containing them): the animated-geometry workload (BASELINE configs[4]
    at C2 scale)."""
    import copy

    s = copy.deepcopy(scene)
    for k, i in enumerate(ids):
        ang = 0.6 * frame + k
        s.prims["trans"][i] += np.array([0.35 * np.cos(ang), 0.2 * np.sin(1.3 * ang), 0.35 * np.sin(ang)])
    for c in range(len(s.clusters)):
        if any(m in ids for m in s.member_idx[s.member_start[c]:s.member_start[c + 1]]):
            s.clusters["lo"][c] -= 0.6
            s.clusters["hi"][c] += 0.6
    return s


def c5_bench(args, local_rank, torch):
    """Animated C2 (8 primitives moving every frame, persistent cascades with
    hysteresis): per frame the scene upload (the grid refit: moved primitives out
    of the lists, BVH refit), relocation and one probe pass, wall clock with the
    stream drained, vs the same with the grid rebuilt every frame."""
    from paper_2007_14394_b200 import api
    from paper_2007_14394_b200.runtime import Device

    base, _ = load_workload("c2")
    rng = np.random.default_rng(5)
    ids = sorted(int(i) for i in rng.choice(len(base.prims), 8, replace=False))
    frames = [animated(base, f, ids) for f in range(1, 11)]
    out = {}
    for mode in ("refit", "rebuild"):
        if mode == "rebuild":
            os.environ["SDFGI_DYNAMIC_MAX"] = "0"
        with Device(local_rank, precision=args.precision) as dev:
            stage = api.ProbeStage(dev, base)
            for p in range(3):
                stage.run_pass(p)
            ms = []
            for f, sc in enumerate(frames):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                stage.set_scene(sc)
                stage.run_pass(3 + f)
                torch.cuda.synchronize()
                ms.append((time.perf_counter() - t0) * 1e3)
            out[mode] = {"ms_per_frame_median": statistics.median(ms[2:]), "ms_first_moving_frame": ms[0]}
        os.environ.pop("SDFGI_DYNAMIC_MAX", None)
    out["workload"] = ("C2 scene, 8 primitives moving every frame, 32x16x32 probes, 256 rays, one pass per "
                       "frame (relocation + update) on persistent cascades")
    out["note"] = ("refit: the moving primitives leave the candidate lists and every on-grid query evaluates "
                   "them; the grid is rebuilt once (frame 1) — rebuild: the grid rebuilt every frame")
    return out


def c4_bench(args, rank, world, local_rank, uid, ext, flush, torch, barrier, dist):
    """BASELINE configs[3] on the same ranks (the slab-sharding workload): C4
    through PASSES passes, same timing rules, fewer steps (one step ~1 s)."""
    from paper_2007_14394_b200 import api
    from paper_2007_14394_b200.runtime import Device

    scene, workload = load_workload("c4")
    with Device(local_rank, rank, world, uid, precision=args.precision) as dev:
        stage = api.ProbeStage(dev, scene)
        runner = StepRunner(dev, stage)
        ext4 = torch.cuda.ExternalStream(dev.stream)
        runner.fresh()
        runner.step()
        steps = max(1, min(args.steps, 2))
        times, _, rays = timed_steps(runner, steps, ext4, flush, torch, barrier)
        ms = max_over_ranks(sum(times) / steps, dist, torch)
        return {"workload": workload, "dtype": args.precision, "n_gpus": world, "steps": steps,
                "ms_per_step": ms, "value": rays / (ms * 1e-3) / 1e9, "unit": UNIT, "rays_per_step": rays,
                "scaling": "strong", "parallelism": f"z-slab x{world}" if world > 1 else "single GPU",
                "primitives": int(len(scene.prims)), "clusters": int(len(scene.clusters))}


def atlas_equal_1gpu(dev, stage, runner, scene, rank, local_rank, dist, torch):
    """SURVEY §8e's correctness test inside the same process group: one fresh step on
    the N ranks (slabs + the NCCL exchange) vs the same step on ONE device (rank 0,
    its own single-rank context): front atlases and probe states bit-identical."""
    from paper_2007_14394_b200 import api
    from paper_2007_14394_b200.runtime import Device

    runner.fresh()
    runner.step()
    got = [dev.atlas(lv, 0) for lv in range(stage.levels)]
    probes = [dev.probes(lv) for lv in range(stage.levels)]
    ok = True
    if rank == 0:
        with Device(local_rank, 0, 1, None, precision=dev.precision) as solo:
            st1 = api.ProbeStage(solo, scene)
            StepRunner(solo, st1).step()
            for lv in range(stage.levels):
                ok = ok and np.array_equal(solo.atlas(lv, 0), got[lv]) and \
                    np.array_equal(solo.probes(lv), probes[lv])
    if dist is not None:
        t = torch.tensor([1 if ok else 0], device="cuda", dtype=torch.int32)
        dist.broadcast(t, src=0)
        ok = bool(t.item())
    return ok


def e2e_run(args, dev, stage, scene, barrier, dist, torch):
    from paper_2007_14394_b200 import api

    # pinned host buffers for the inputs (fresh probes) and the result (atlas)
    n = int(np.prod(scene.cascade.res))
    t = dev.oct_res + 2
    probes_pin = torch.empty(n * scene_io.PROBE_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
    probes_host = probes_pin.numpy().view(scene_io.PROBE_DTYPE)
    stage.reset()
    probes_host[:] = dev.probes(0)  # the fresh volume (makeCascade state)
    atlas_pin = torch.empty(n * t * t * 3, dtype=torch.float32, pin_memory=True)
    atlas_host = atlas_pin.numpy().reshape(n, t, t, 3)
    scene_bytes = (scene.prims.nbytes + scene.clusters.nbytes + scene.member_start.nbytes +
                   scene.member_idx.nbytes + scene.lights.nbytes + 24)
    h2d = int(scene_bytes + probes_host.nbytes)
    d2h = int(atlas_host.nbytes)
    steps = max(1, min(args.steps, 5))
    total, rays = 0.0, 0
    for i in range(steps + 1):
        barrier()
        t0 = time.perf_counter()
        dev.upload_scene(scene)
        dev.reset_probes(0)  # fresh volume: zero atlases (makeCascade)
        dev.upload_probes(0, probes_host)
        r = 0
        for p in range(PASSES):  # relocation + update queued (sdfgi_probe_stage_async) + swap
            dev.probe_stage_async(p, stage.cfg)
            dev.swap()
        r = int(dev.probe_stage_collect()[1]["rays_traced"].sum())
        dev.atlas(0, 0, out=atlas_host)  # straight into the pinned buffer
        dt = time.perf_counter() - t0
        if i > 0:  # first iteration is a warm-up
            total += dt
            rays = r
    if dist is not None:
        tt = torch.tensor([total], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    return rays * steps / total / 1e9, h2d, d2h


def gather_bench(args, dev, stage, scene, torch, ext, flush):
    """C3: 1920x1080 gather on the C2 volume after its 3 bounces. The
    G-buffer is the gather's input (rendered once on the device, not timed, as the
    reference's t_gbuffer is separate, pipeline.hpp:155-159); each timed frame runs
    the whole gather (downsample, selection, tile visibility + shadePixelGI, resolve
    with history, Contact GI) against the front atlas, L2 flushed before it."""
    w, h = 1920, 1080
    cfg = stage.cfg
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    dev.render_gbuffer(scene.camera, w, h, cfg)
    e1.record(ext)
    e1.synchronize()
    gbuffer_ms = e0.elapsed_time(e1)
    dev.reset_history()
    tasks, vs, cs = dev.gather(0, cfg, stats=True)
    for f in range(1, args.warmup + 1):
        dev.gather(f, cfg)
    _, _, ps = dev.compose(cfg, stats=True, download=False)
    times, stages, ctimes = [], [], []
    for k in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0.record(ext)
        dev.gather(args.warmup + 1 + k, cfg)
        e1.record(ext)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        stages.append(dev.last_gather_ms())
        # composeFrame (f1, pipeline.hpp:209) on this frame's indirect image: device
        # time from the call's own events (the image stays in HBM)
        ctimes.append(dev.compose(cfg, download=False)[1])
    st = np.median(np.array(stages), axis=0)
    res = {
        "config": "C3: 1920x1080, frame with history, C2 scene and volume after 3 bounces",
        "ms_per_frame": float(np.median(times)),
        "stage_ms": {"downsample_select": st[0], "tiles_visibility_shadePixelGI": st[1], "resolve": st[2],
                     "contact_gi": st[3]},
        "compose_ms": float(np.median(ctimes)),
        "compose_shadow_traces_per_pixel": int(ps["shadow_traces"]) / (w * h),
        "gbuffer_ms_input": gbuffer_ms,
        "visibility_tasks": int(tasks),
        "visibility_traces_per_pixel": int(vs["visibility_traces"]) / (w * h),
        "contact_rays_per_pixel": int(cs["sphere_traces"]) / (w * h),
        "contact_sdf_queries_per_pixel": int(cs["sdf_queries"]) / (w * h),
    }
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_gather_baseline()
    return res


def cpu_gather_baseline():
    """The reference gather (pipeline.hpp:161-207) on all host threads at 480x270
    (1/16 of the 1080p pixels; 3 probe passes of 32 rays seed the atlas), frame 1."""
    exe = ref_binary()
    if exe is None:
        return None
    threads = cpu_threads()
    cmd = [exe, "gather", C2_PATH, os.devnull, "--passes", "1", "--nrays", "32", "--threads", str(threads),
           "--size", "480", "270", "--gather-frames", "2", "--no-dump"]
    r = subprocess.run(cmd, capture_output=True, text=True, check=True)
    out = json.loads(r.stdout)
    f = out["frames"][1]
    ms = f["visibility_ms"] + f["resolve_ms"] + f["contact_ms"]
    cms = f.get("compose_ms")
    return {"ms_per_frame_sample": ms, "ms_per_frame_1080p_scaled": ms * 16, "cores": threads,
            "compose_ms_1080p_scaled": None if cms is None else cms * 16,
            "kind": "reference", "sample": "480x270 (1/16 of 1080p pixels), frame with history; scaled x16"}


def cpu_baseline(rays_full_step):
    threads = cpu_threads()
    stride = int(os.environ.get("SDFGI_CPU_STRIDE", str(CPU_STRIDE["c2"])))
    res, kind = cpu_reference_sample(stride, threads)
    if res is None:
        return {"value": None, "unit": UNIT, "cores": threads, "kind": "reference", "sample": kind}
    rays, secs = res[0]
    return {
        "value": rays / secs / 1e9,
        "unit": UNIT,
        "cores": threads,
        "kind": "reference",
        "binary": kind,
        "sample": f"C2 scene, 3 passes, every {stride}th probe ({rays} rays, {secs:.2f} s; relocation time "
                  f"scaled by 1/{stride}); full step = {rays_full_step} rays",
    }


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = cpu_threads()
    stride = int(os.environ.get("SDFGI_CPU_STRIDE", str(CPU_STRIDE[args.config])))
    res, kind = cpu_reference_sample(stride, threads, reps=args.warmup + args.steps, sdfs=workload_sdfs(args.config))
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": kind}))
        return
    timed = res[args.warmup:]
    rays = sum(r for r, _ in timed)
    secs = sum(s for _, s in timed)
    value = rays / secs / 1e9
    sample = (f"{args.config.upper()} scene, 3 passes, every {stride}th probe per step ({timed[0][0]} rays/step), "
              f"{threads} threads, relocation time scaled by 1/{stride}")
    print(json.dumps({
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": secs / len(timed) * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic (deterministic {args.config.upper()} scene)",
        "config": {"workload": WORKLOADS[args.config],
                   "path": "reference CPU probe stage, pipeline.hpp:108-151 (updateProbePositions + "
                           "parallelFor(updateProbe)), all host threads",
                   "sample_stride": stride, "binary": kind},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: re-run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous)."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--config", default="c2", choices=["c2", "c4"],
                    help="c2: the headline workload (BASELINE configs[1]); c4: configs[3]")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gather", action="store_true", help="skip the C3 1080p gather measurement")
    ap.add_argument("--no-alt", action="store_true", help="skip the other-precision measurement")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 sub-measurement of a c2 run")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
