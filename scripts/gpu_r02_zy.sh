#!/bin/bash
# power / clock vs item order (DRAM locality) for the full pass and the no-arithmetic floor
mkdir -p gpurun_out
O=gpurun_out/power_order.jsonl
for v in base floor; do
  if [ $v = base ]; then L=; else L=variants/$v.so; fi
  for o in 0 1 2; do
    SSB_ORDER=$o SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py config4 | sed "s/\"config\"/\"var\": \"$v order $o\", \"config\"/" >> $O 2>&1
  done
  SSB_SNAKE=0 SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py config4 | sed "s/\"config\"/\"var\": \"$v nosnake\", \"config\"/" >> $O 2>&1
done
grep '^{' $O | cut -c1-200
