#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/power.jsonl
timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
SUBSURF_B200_LIB=variants/w16c1.so timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
SUBSURF_B200_LIB=variants/nofillpass.so timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
timeout 300 python scripts/power_probe.py config1 >> $O 2>&1
cat $O
