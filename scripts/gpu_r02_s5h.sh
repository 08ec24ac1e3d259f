#!/bin/bash
# session 5: flakiness check -- the whole GPU suite five times back to back (-x, as the driver runs it)
mkdir -p gpurun_out
for i in 1 2 3 4 5; do
  timeout 1500 python -m pytest tests -m gpu -q -x -W always > gpurun_out/s5h_suite$i.log 2>&1
  echo "suite $i rc=$? $(tail -1 gpurun_out/s5h_suite$i.log)" | tee -a gpurun_out/s5h_summary.txt
done
grep -l "failed once" gpurun_out/s5h_suite*.log
nvidia-smi --query-compute-apps=pid,used_memory --format=csv
