#!/bin/bash
# session 5: the whole GPU suite (no -x, durations), the bench-dist test carrying the watchdog
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/s5d_suite.log 2>&1
tail -30 gpurun_out/s5d_suite.log
nvidia-smi --query-compute-apps=pid,used_memory --format=csv
