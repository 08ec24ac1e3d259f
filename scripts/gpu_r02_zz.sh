#!/bin/bash
# power: the no-arithmetic floor with and without the l+-1 row copies (L2-hit traffic)
mkdir -p gpurun_out
O=gpurun_out/power_nolpm.jsonl
rm -f $O
for rep in 1 2; do
  for v in floor floornolpm; do
    SUBSURF_B200_LIB=variants/$v.so timeout 300 python scripts/power_probe.py config4 | sed "s/\"config\"/\"var\": \"$v\", \"config\"/" >> $O 2>&1
  done
done
grep '^{' $O | cut -c1-200
