"""Join an ncu SASS source page (CSV, one kernel) with nvdisasm line info of the same
kernel: stall samples, executed instructions and active threads per source line.
usage: python scripts/sass_lines.py <sass.csv> <nvdisasm -c -gi output> <mangled kernel> [n]"""
import collections
import csv
import re
import sys

sass_csv, dis, fn = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{fn}:"))
loc = {}
cur, outer = "?", "?"
fresh = True  # the first //## File line after an instruction is the innermost location
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//-----"):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        if fresh:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            outer = f"{m.group(3).split('/')[-1]}:{m.group(4)}" if m.group(3) else cur
        fresh = False
        continue
    fresh = True
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m:
        loc[int(m.group(1), 16)] = (cur, outer)
rows = list(csv.reader(open(sass_csv)))
h = rows[0]
col = {c: i for i, c in enumerate(h)}


def num(x):
    try:
        return float(x)
    except ValueError:
        return None


data = [r for r in rows[1:] if len(r) == len(h) and num(r[col["Instructions Executed"]]) is not None]
base = int(data[0][col["Address"]], 16)
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in data:
    off = int(r[col["Address"]], 16) - base
    key = loc.get(off, ("?", "?"))[0]
    a = agg[key]
    a[0] += num(r[col["Warp Stall Sampling (All Samples)"]]) or 0
    a[1] += num(r[col["Instructions Executed"]]) or 0
    a[2] += num(r[col["Thread Instructions Executed"]]) or 0
ts = sum(a[0] for a in agg.values()) or 1
te = sum(a[1] for a in agg.values()) or 1
print(f"{'line':28s} {'stall%':>7s} {'inst%':>7s} thr/inst")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k:28s} {a[0] / ts * 100:7.2f} {a[1] / te * 100:7.2f} {a[2] / max(a[1], 1):5.1f}")
