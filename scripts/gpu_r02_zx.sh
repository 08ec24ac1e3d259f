#!/bin/bash
# data-movement floor of the SOR pass under the power cap (timing-only variant: no arithmetic)
mkdir -p gpurun_out
O=gpurun_out/power_floor.jsonl
for rep in 1 2; do
  for v in base floor; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py config4 | sed "s/\"config\"/\"var\": \"$v\", \"config\"/" >> $O 2>&1
  done
done
grep '^{' $O | cut -c1-200
