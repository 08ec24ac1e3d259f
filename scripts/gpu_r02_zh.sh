#!/bin/bash
# SOR try_wait suspend-time hints under the power cap (power_probe: 3000-sweep config-4 loops)
mkdir -p gpurun_out
O=gpurun_out/power_susp.jsonl
for rep in 1 2; do
  for v in base sus200 sus2000 sus20000 sus1000000; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
  done
done
cat $O
