#!/bin/bash
# power: two of the ten 8-byte shared-memory operand loads dropped (timing only, wrong values)
mkdir -p gpurun_out
O=gpurun_out/power_ldsx.jsonl
rm -f $O
for rep in 1 2 3; do
  for v in base ldsx; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py config4 2>&1 | tail -1 | sed "s/\"config\"/\"var\": \"$v\", \"config\"/" >> $O
  done
done
cut -c1-220 $O
