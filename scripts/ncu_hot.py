"""Summarise an ncu source page (SASS): stall share, instruction share and active
threads per instruction of the hottest instructions, plus per-source-line totals."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Address" in r or "# Address" in r)
start = rows.index(hdr) + 1
data = [r for r in rows[start:] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
ss = col.get("Warp Stall Sampling (All Samples)")
ie = col.get("Instructions Executed")
it = col.get("Thread Instructions Executed")
src = col.get("Source")
f = lambda r, i: float(r[i]) if i is not None and r[i] not in ("", "-") else 0.0
ts = sum(f(r, ss) for r in data) or 1
te = sum(f(r, ie) for r in data) or 1
tt = sum(f(r, it) for r in data)
print(f"samples {ts:.0f} inst {te:.3g} threads/inst {tt / te:.2f}")
for r in sorted(data, key=lambda r: -f(r, ss))[:n]:
    e = f(r, ie)
    print(f"{f(r, ss) / ts * 100:5.1f}% stall {e / te * 100:5.2f}% inst thr={f(r, it) / e if e else 0:4.1f}  {r[src][:90]}")
