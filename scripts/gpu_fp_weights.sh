#!/bin/bash
# One gpurun call: the measured FP instruction weights of the shading kernels and the
# executed FP instructions of every update kernel (scripts/measure_fp_ops.py), both
# precisions -> gpurun_out/fp_weights_<prec>.json (+ the ncu CSVs).
mkdir -p gpurun_out
M=$(python3 -c "import sys; sys.argv=['x']; exec(open('scripts/measure_fp_ops.py').read().split('def run')[0]); print(METRICS)")
for prec in f64 f32; do
  python scripts/measure_fp_ops.py run $prec gpurun_out/fp_counts_$prec.json
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp_ops_$prec.csv \
      python scripts/measure_fp_ops.py run $prec /dev/null > /dev/null 2>&1
  python scripts/measure_fp_ops.py summarize $prec gpurun_out/fp_counts_$prec.json gpurun_out/fp_ops_$prec.csv \
      gpurun_out/fp_weights_$prec.json
done
