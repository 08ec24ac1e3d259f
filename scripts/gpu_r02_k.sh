#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/power_k.jsonl
for r in 1 2; do
timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
SUBSURF_B200_LIB=variants/nores.so timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
done
cat $O
