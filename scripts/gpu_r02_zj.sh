#!/bin/bash
# j-wavefront one-sweep kernel (kernel 7) vs the two-pass under the power cap (config 4)
mkdir -p gpurun_out
O=gpurun_out/power_kwave.jsonl
for v in "tma base" "kwave kw16" "kwave kw16l3" "kwave base"; do
  set -- $v
  if [ $2 = base ]; then L=; else L=variants/$2.so; fi
  SUBSURF_B200_LIB=$L SUBSURF_KERNEL=$1 timeout 300 python scripts/power_probe.py config4 | sed "s/\"config\"/\"var\": \"$2\", \"config\"/" >> $O 2>&1
done
cat $O
