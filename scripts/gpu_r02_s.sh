#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/power_s.jsonl
for r in 1 2; do
timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
SUBSURF_B200_LIB=variants/fw4.so timeout 300 python scripts/power_probe.py config4 | sed 's/"config"/"variant": "fw4", "config"/' >> $O 2>&1
done
cat $O
