#!/bin/bash
# One gpurun call: ncu launch lists of a full C2 step + G-buffer + gather
# (scripts/profile_step.py) and a `--set full` capture of the hot update kernels
# on a C2 pass (scripts/profile_update.py), summarised on the box into
# gpurun_out/ncu_step_<prec>.json (the .ncu-rep files are too big to bring back).
# usage: bash scripts/gpu_profile_round.sh [f64 f32]
mkdir -p gpurun_out
for prec in ${@:-f64 f32}; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio \
      --clock-control none --csv --log-file gpurun_out/step_launches_$prec.csv \
      python scripts/profile_step.py $prec > gpurun_out/ncu_launch_$prec.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:'k_trace|k_shade|k_convolve|k_hit' \
      -f -o /tmp/full_$prec python scripts/profile_update.py $prec 1 1 > gpurun_out/ncu_full_$prec.log 2>&1
  python scripts/summarize_ncu.py gpurun_out/step_launches_$prec.csv /tmp/full_$prec.ncu-rep \
      gpurun_out/ncu_step_$prec.json > gpurun_out/summ_$prec.log 2>&1
done
