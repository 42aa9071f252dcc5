"""Summaries committed under profiles/: per-kernel share of a step from the launch
list, and the key metrics of each full capture."""
import csv
import json
import subprocess
import sys
from collections import defaultdict

launches, full, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = defaultdict(lambda: defaultdict(float))
count = defaultdict(set)
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    try:
        per[name][r[mi]] += float(r[vi].replace(",", ""))
    except ValueError:
        continue
    count[name].add(r[ii])
tot = sum(v["gpu__time_duration.sum"] for v in per.values())
summary = {"launch_list": {}, "total_kernel_ms": tot / 1e6}
for name, v in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    n = len(count[name])
    summary["launch_list"][name] = {
        "launches": n, "ms": v["gpu__time_duration.sum"] / 1e6, "share": v["gpu__time_duration.sum"] / tot,
        "dram_bytes_per_launch": (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / max(n, 1),
        "active_threads_per_inst": v.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0) / max(n, 1),
    }
raw = subprocess.run(["ncu", "-i", full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size"]
idx = {w: h.index(w) for w in want if w in h}
units = rr[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
summary["full_captures"] = []
for r in rr[2:]:
    if len(r) != len(h):
        continue
    cap = {}
    for w, i in idx.items():
        u = units[i]
        if u in SCALE:  # normalised: bytes and nanoseconds
            cap[w] = repr(float(r[i].replace(",", "")) * SCALE[u])
        else:
            cap[w] = r[i]
    summary["full_captures"].append(cap)
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary["launch_list"], indent=1)[:3000])
for c in summary["full_captures"]:
    print({k: c[k] for k in list(c)[:1]}, {k.split("__")[-1][:40]: c[k] for k in list(c)[1:]})
