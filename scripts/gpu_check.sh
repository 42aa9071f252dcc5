#!/bin/bash
# One gpurun call for an iteration: GPU tests (summary lines), a short bench
# (headline numbers), and the ncu launch list of one C2 step + gather (top kernels).
# usage: bash scripts/gpu_check.sh <tag> [pytest -k expr]
tag=${1:-x}
mkdir -p gpurun_out
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
python -m pytest tests -m gpu -q -x -s -p no:cacheprovider $K 2>&1 | grep -E "C2 pass|C3 frame|passed|failed|Error|assert" | head -30
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c4 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python3 - "$tag" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
g = d["gather_c3"]
print(f"step {d['ms_per_step']:.2f} ms  {d['value']:.4f} Grays/s  e2e {d['e2e']['value']:.4f}  f32 {d['alt_precision']['ms_per_step']:.2f} ms  "
      f"gather {g['ms_per_frame']:.2f} ms {g['stage_ms']}  roofline {d['roofline']['frac']:.4f}")
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$tag.csv python scripts/profile_step.py f64 > /dev/null 2>&1
python scripts/launch_times.py gpurun_out/launch_$tag.csv 2>/dev/null | head -14
