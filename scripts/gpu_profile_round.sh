#!/bin/bash
# One gpurun call: ncu launch lists of a full C2 step + G-buffer + gather
# (scripts/profile_step.py) and a `--set full` capture of the update kernels of C2
# pass 1 (N rays per probe, bounce lookups on: scripts/profile_pass.py, the 9
# launches after pass 0's 9), summarised on the box into gpurun_out/ncu_step_<prec>.json
# (the .ncu-rep files are too big to bring back).
# usage: bash scripts/gpu_profile_round.sh [f64 f32]
mkdir -p gpurun_out
for prec in ${@:-f64 f32}; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio \
      --clock-control none --csv --log-file gpurun_out/step_launches_$prec.csv \
      python scripts/profile_step.py $prec > gpurun_out/ncu_launch_$prec.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:'k_trace|k_shade|k_convolve|k_hit' \
      --launch-skip 9 --launch-count 9 -f -o /tmp/full_$prec python scripts/profile_pass.py $prec 2 \
      > gpurun_out/ncu_full_$prec.log 2>&1
  python scripts/summarize_ncu.py gpurun_out/step_launches_$prec.csv /tmp/full_$prec.ncu-rep \
      gpurun_out/ncu_step_$prec.json > gpurun_out/summ_$prec.log 2>&1
  cp /tmp/full_$prec.ncu-rep gpurun_out/ 2>/dev/null
done
