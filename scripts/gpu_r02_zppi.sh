#!/bin/bash
# planes per item 16 (default) / 32 / 64 under the power cap on configs 4, 2, 1
mkdir -p gpurun_out
O=gpurun_out/power_ppi2.jsonl; rm -f $O
for c in config4 config2 config1; do
  for rep in 1 2; do for v in base ppi32 ppi64; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py $c 2>&1 | tail -1 | sed "s/\"config\"/\"var\": \"$v\", \"config\"/" >> $O
  done; done
done
cut -c1-160 $O
