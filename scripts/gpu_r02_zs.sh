#!/bin/bash
# power sensitivity of the SOR pass to its FP64 work (timing-only variants, wrong results)
mkdir -p gpurun_out
O=gpurun_out/power_fp64b.jsonl
for rep in 1 2; do
  for v in base sx4 sx8 sx12; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py config4 | sed "s/\"config\"/\"var\": \"$v\", \"config\"/" >> $O 2>&1
  done
done
cat $O
