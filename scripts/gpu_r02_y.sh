#!/bin/bash
mkdir -p gpurun_out
if timeout 600 python scripts/step_launch_list.py config4 2 > gpurun_out/sll.log 2>&1; then
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_step_c4.csv python scripts/step_launch_list.py config4 2 > gpurun_out/ncu_sll.log 2>&1
fi
tail -2 gpurun_out/sll.log; ls -la gpurun_out/launches_step_c4.csv
